# TF32 TMA-store epilogue: tests + full TF32 probe:  gpurun --timeout 1500 -- 'bash tools/gpu_r02t.sh'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r02t
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_large.py tests/test_cli.py -q -k "tf32" > gpurun_out/r02t/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02t/pytest.log | cut -c1-400
timeout 600 python tools/tf32_probe.py 2048 4096 8192 > gpurun_out/r02t/tf32_probe.log 2>&1; echo "probe rc=$?"; cat gpurun_out/r02t/tf32_probe.log
