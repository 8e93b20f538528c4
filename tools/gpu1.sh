set -x
nproc; nvidia-smi -L
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -20
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -40
timeout 600 python tools/gpu_probe.py 2>&1 | tail -40
