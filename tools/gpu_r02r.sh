# TF32 stream-K restricted to long K: tests + A/B + full TF32 probe
#   gpurun --timeout 1500 -- 'bash tools/gpu_r02r.sh'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r02r
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_large.py -q -k tf32 > gpurun_out/r02r/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02r/pytest.log | cut -c1-300
timeout 600 python tools/tf32_sk_check.py > gpurun_out/r02r/tf32_sk.log 2>&1; echo "sk check rc=$?"; grep -v "^{" gpurun_out/r02r/tf32_sk.log | grep -v "^ *$" | cut -c1-200
timeout 600 python tools/tf32_probe.py 2048 4096 8192 > gpurun_out/r02r/tf32_probe.log 2>&1; echo "probe rc=$?"; grep "best" gpurun_out/r02r/tf32_probe.log
