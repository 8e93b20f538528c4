cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_ptxgen.py -q -x 2>&1 | grep -E "AssertionError|assert|gemm\||\(" | head -20 | cut -c1-1500
