# Stream-K first light + A/B, then full-search shard 5 and the full GPU suite:
#   gpurun --timeout 5400 -- 'bash tools/gpu_r02k.sh'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r02k
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "stream_k or split_k" > gpurun_out/r02k/sk_pytest.log 2>&1; echo "sk pytest rc=$?"; tail -15 gpurun_out/r02k/sk_pytest.log | cut -c1-300
timeout 1500 python tools/sk_probe.py --per-tile 8 --shapes 2048x2048x2048,8192x256x8192,1024x1024x1024 > gpurun_out/r02k/sk_probe.log 2>&1; echo "sk probe rc=$?"
cut -c1-3000 gpurun_out/r02k/sk_probe.log
FS_TIMEOUT=${FS_T:-2800} bash tools/gpu_fullsearch_4096.sh 710510 142098
