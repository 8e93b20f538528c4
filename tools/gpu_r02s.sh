# Validation of HEAD after the TF32 stream-K change:  gpurun --timeout 2400 -- 'bash tools/gpu_r02s.sh'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r02s
export KTC_SEGV_TRACE=1
timeout 1800 python -m pytest tests/ -q -m gpu > gpurun_out/r02s/pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02s/pytest.log | cut -c1-300
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r02s/bench_default.log 2>&1; echo "bench default rc=$?"
tail -1 gpurun_out/r02s/bench_default.log | cut -c1-300
