# Round-end validation on a B200 (run under gpurun from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 2700 -- 'bash tools/gpu_validate.sh'
# GPU test suite, smoke(), the bench line and the reference arm; logs in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
export KTC_SEGV_TRACE=1
timeout 1800 python -m pytest tests/ -q -m gpu -x > gpurun_out/validate_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/validate_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/validate_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/validate_bench.log | cut -c1-400
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/validate_bench_ref.log 2>&1
tail -1 gpurun_out/validate_bench_ref.log | cut -c1-300
