# Conv generator pair-register change: bit-parity vs NVRTC, conv parity, bench
#   gpurun --timeout 2400 -- 'bash tools/gpu_r02y.sh'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r02y
timeout 1200 python -m pytest tests/test_gpu_ptxgen.py tests/test_gpu_parity.py tests/test_gpu_parity_large.py tests/test_gpu_ffma2.py -q -k "conv or ptx or ffma2" > gpurun_out/r02y/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02y/pytest.log | cut -c1-300
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02y/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r02y/bench.log | cut -c1-300
timeout 900 python bench.py --steps 20 --warmup 5 --no-tuned --no-cpu > gpurun_out/r02y/bench2.log 2>&1; echo "bench2 rc=$?"
tail -1 gpurun_out/r02y/bench2.log | cut -c1-300
