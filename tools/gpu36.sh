cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export KTC_SEGV_TRACE=1
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/r36_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r36_pytest.log
KTC_TRACE=1 timeout 600 python tools/e2e_probe.py 2>&1 | grep -E "job|same|tune: backends|build inputs|destroy" | head -30
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r36_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r36_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['value_warm_cache'], d['e2e'], d['clocks']); print(d['roofline']); t=d['tuned']; print({f:(round(v['gflops']),round(v['frac'],3)) for f,v in t['conv'].items()}, t.get('sgemm_2048',{}).get('gflops'), t.get('tf32_2048',{}).get('gflops')); print(d['cpu_baseline'])"
