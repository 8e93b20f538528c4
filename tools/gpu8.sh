cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -5
export KTC_CACHE_DIR=/tmp/ktc_ab
timeout 600 python tools/gemm_ab.py --size 2048 --fraction 512 --out gpurun_out/ab_d1o1.json 2>&1 | tail -2
KTC_GEMM_DBUF_MAX=0 KTC_GEMM_OCC=0 timeout 600 python tools/gemm_ab.py --size 2048 --fraction 512 --out gpurun_out/ab_d0o0.json 2>&1 | tail -2
KTC_GEMM_OCC=0 timeout 600 python tools/gemm_ab.py --size 2048 --fraction 512 --out gpurun_out/ab_d1o0.json 2>&1 | tail -2
KTC_GEMM_DBUF_MAX=0 timeout 600 python tools/gemm_ab.py --size 2048 --fraction 512 --out gpurun_out/ab_d0o1.json 2>&1 | tail -2
unset KTC_CACHE_DIR
timeout 900 python bench.py --steps 5 --warmup 3 2>&1 | tail -1
