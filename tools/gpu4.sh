cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -25
timeout 600 python bench.py --steps 5 --warmup 3 --no-tuned 2>&1 | tail -3
timeout 2400 python tools/tune_sweep.py --tag r01 --gemm-fraction 0.002 --tf32 2>&1 | tail -20
