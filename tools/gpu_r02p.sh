# SGEMM host-switch A/B at 2048^3 (double-buffer threshold, register budget):
#   gpurun --timeout 2400 -- 'bash tools/gpu_r02p.sh'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r02p
timeout 2000 python tools/sk_probe.py --per-tile 10 --shapes 2048x2048x2048 \
  --variants "dbuf:;nodbuf:KTC_GEMM_DBUF_MAX=0;occ0:KTC_GEMM_OCC=0;dbuf160k:KTC_GEMM_DBUF_MAX=163840" > gpurun_out/r02p/ab.log 2>&1; echo "ab rc=$?"
python - <<'PY'
import json
d=json.load(open('gpurun_out/sk_probe_2048x2048x2048.json'))
for k,v in sorted(d['per_tile'].items(), key=lambda kv: -max(x['tflops'] for x in kv[1].values())):
    print(k, {m: round(x['tflops'],1) for m,x in v.items()})
print('not verified', {m: len(r) for m,r in d['not_verified'].items()}, 'errors', list(d['errors']))
PY
