# pass d: prune-probe check + 4096^3 full-search rate probe + bench.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r02d
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "prune or sharded" > gpurun_out/r02d/prune.log 2>&1; echo "prune tests rc=$?"; tail -2 gpurun_out/r02d/prune.log
timeout 900 python tools/gemm_full_search.py --size 4096 --start 400000 --count 4000 --prune 2 > gpurun_out/r02d/fs_probe.log 2>&1; echo "fs probe rc=$?"; tail -1 gpurun_out/r02d/fs_probe.log | cut -c1-400
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r02d/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r02d/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['value_warm_cache'], d['configs4_gemm4096']['value'], d['roofline']['frac'])"
