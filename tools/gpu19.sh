cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export KTC_SEGV_TRACE=1
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/r19_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r19_pytest.log
timeout 600 python tools/tf32_repro.py 4 > gpurun_out/tf32_repro.log 2>&1; echo "repro rc=$?"; tail -5 gpurun_out/tf32_repro.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r19_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r19_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['value_warm_cache'], d['e2e']); print(json.dumps(d['tuned'])[:1500]); print(d['roofline'])"
