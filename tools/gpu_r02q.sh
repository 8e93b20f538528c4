# TF32 stream-K: coalesced partials, release/acquire publish, cluster-count sweep
#   gpurun --timeout 900 -- 'bash tools/gpu_r02q.sh'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r02q
for g in none 56 60 64 66 68 70 72 74; do
  if [ "$g" = none ]; then unset KTC_SK_G; else export KTC_SK_G=$g; fi
  KTC_TF32_SK=1 timeout 120 python -c "
import sys; sys.path.insert(0,'.')
import paper_1703_06503_b200 as pkg
be=pkg.CudaBackend(0)
for cfg in (dict(BN=256,BK=64,STAGES=3,CG=2), dict(BN=256,BK=32,STAGES=3,CG=2)):
    r=be.evaluate(pkg.gemm_request(2048,2048,2048,cfg,tf32=True,reps=10))
    print('G=$g', cfg, r.status, r.verification, r.time_ms if r.ok else r.message[:100])
" 2>&1 | tail -2
done
unset KTC_SK_G
timeout 600 python tools/tf32_sk_check.py > gpurun_out/r02q/tf32_sk.log 2>&1; echo "sk check rc=$?"; grep -v "^{" gpurun_out/r02q/tf32_sk.log | grep -v "^$" | cut -c1-200
