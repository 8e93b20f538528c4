cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/ -q -m gpu 2>&1 | tail -15
timeout 600 python tools/tune_sweep.py --tag tf32 --skip-conv --skip-gemm --tf32 2>&1 | tail -3
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_verify.csv python tools/profile_winners.py conv3 > /dev/null 2>&1
grep -E "verify|conv2d" gpurun_out/launches_verify.csv | head
timeout 900 python bench.py --steps 5 --warmup 3 2>&1 | tail -2
