cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1500 python tools/split_probe.py --top 150 --shapes 2048x2048x2048,1024x1024x1024,8192x256x8192,4096x4096x4096 > gpurun_out/split_probe.log 2>&1; echo rc=$?
cat gpurun_out/split_probe.log | cut -c1-2000
timeout 600 python -m pytest tests/test_gpu_ptxgen.py -q -x 2>&1 | tail -2
