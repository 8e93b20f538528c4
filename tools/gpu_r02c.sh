# Round-2 pass c: isolated-worker fault tests, memcheck negative control,
# e2e after the pinned pool + module reaper.  gpurun --timeout 2400 -- 'bash tools/gpu_r02c.sh'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r02c gpurun_out/sanitizer
timeout 900 python -m pytest tests/test_gpu_faults.py tests/test_gpu_custom_kernel.py -q > gpurun_out/r02c/faults.log 2>&1; echo "faults rc=$?"; tail -3 gpurun_out/r02c/faults.log
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 600 $CS --tool memcheck --leak-check no --print-limit 5 python tools/sanitize_configs.py --control \
    > gpurun_out/sanitizer/memcheck_control.log 2>&1
echo "memcheck control rc=$?"; grep -m3 "Invalid\|ERROR SUMMARY\|control row" gpurun_out/sanitizer/memcheck_control.log
KTC_TRACE=1 timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r02c/bench.log 2> gpurun_out/r02c/bench.err; echo "bench rc=$?"
tail -1 gpurun_out/r02c/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'], d['value_warm_cache'], d.get('configs4_gemm4096'))"
