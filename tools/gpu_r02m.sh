# TF32 stream-K first light:  gpurun --timeout 1500 -- 'bash tools/gpu_r02m.sh'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r02m
timeout 900 python tools/tf32_sk_check.py > gpurun_out/r02m/tf32_sk.log 2>&1; echo "sk rc=$?"
cat gpurun_out/r02m/tf32_sk.log | cut -c1-300
if grep -q "2048x2048x2048 {'BN': 256, 'BK': 64, 'STAGES': 3, 'CG': 2} \['ok', 'pass'" gpurun_out/r02m/tf32_sk.log; then
  timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_large.py -q -k tf32 > gpurun_out/r02m/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02m/pytest.log
  timeout 600 python tools/tf32_probe.py 2048 > gpurun_out/r02m/tf32_probe.log 2>&1; cat gpurun_out/r02m/tf32_probe.log
fi
