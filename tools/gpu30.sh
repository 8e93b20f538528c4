cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "prune" 2>&1 | tail -3
timeout 1500 python tools/gemm_sweeps.py --sample 2048 --skip-shapes --prune 2.0 2>&1 | cut -c1-400
timeout 600 python tools/tf32_probe.py 2048 4096 8192 2>&1 | tail -16
