cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/cublas_ref.py --out gpurun_out/cublas_sgemm.json 2>&1 | tail -4
timeout 900 python bench.py --steps 5 --warmup 3 --no-tuned > gpurun_out/r11_bench.log 2>&1; tail -1 gpurun_out/r11_bench.log | cut -c1-200; tail -1 gpurun_out/r11_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['value_warm_cache'], d['e2e'])"
timeout 600 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -2
