cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export KTC_SEGV_TRACE=1
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/r20_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r20_pytest.log
timeout 600 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1; echo "e2e rc=$?"; cat gpurun_out/e2e_probe.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r20_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r20_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['value_warm_cache'], d['e2e']); print(d['roofline']); print(d['tuned'].get('sgemm_2048'))"
