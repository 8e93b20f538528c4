cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -15
timeout 600 python bench.py --steps 3 --warmup 3 --no-tuned 2>&1 | tail -5
timeout 900 python tools/tune_sweep.py --tag probe --filters 3 --conv-fraction 0.25 --gemm-fraction 0.0005 2>&1 | tail -20
