cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/r28_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r28_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r28_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r28_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['value_warm_cache'], d['e2e'], d['clocks']); print(d['roofline']); t=d['tuned']; print({f:(round(v['gflops']),round(v['frac'],3)) for f,v in t['conv'].items()}, t.get('sgemm_2048',{}).get('gflops'), t.get('tf32_2048',{}).get('gflops')); print(d['cpu_baseline'])"
