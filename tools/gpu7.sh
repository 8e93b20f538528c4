cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "verifier or smoke or reference_small" 2>&1 | tail -3
timeout 900 python bench.py --steps 5 --warmup 3 2>&1 | tail -1
timeout 2700 python tools/gemm_sweeps.py 2>&1 | tail -20
