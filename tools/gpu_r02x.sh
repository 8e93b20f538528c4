# TF32 stream-K with double-buffered TMEM + TMA-store output: tests, check, trace, A/B
#   gpurun --timeout 1200 -- 'bash tools/gpu_r02x.sh'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r02x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "tf32" > gpurun_out/r02x/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02x/pytest.log | cut -c1-300
timeout 600 python tools/tf32_sk_check.py > gpurun_out/r02x/tf32_sk.log 2>&1; echo "sk check rc=$?"; grep -v "^{" gpurun_out/r02x/tf32_sk.log | grep -v "^ *$" | grep -v "CG': 1}" | cut -c1-200
for sk in 0 2; do
  KTC_TF32_SK=$sk timeout 120 python -c "
import sys; sys.path.insert(0,'.')
import paper_1703_06503_b200 as pkg
be=pkg.CudaBackend(0)
for cfg in (dict(BN=256,BK=64,STAGES=3,CG=2), dict(BN=256,BK=32,STAGES=3,CG=2), dict(BN=128,BK=64,STAGES=3,CG=2), dict(BN=256,BK=32,STAGES=3,CG=1)):
    r=be.evaluate(pkg.gemm_request(2048,2048,2048,cfg,tf32=True,reps=10))
    print('SK=$sk', cfg, r.status, r.verification, r.time_ms if r.ok else r.message[:100])
" 2>&1 | tail -4
done
timeout 300 python tools/tf32_sk_trace.py 2>&1 | grep -E "median|max per|ok pass"
