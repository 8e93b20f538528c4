# Re-validation of HEAD on one B200 after the isolated backend / split-K tail
# changes:  gpurun --timeout 2700 -- 'bash tools/gpu_r02e.sh'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
export KTC_SEGV_TRACE=1
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/r02e_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r02e_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python tools/tail_ab.py > gpurun_out/r02e_tail_ab.json 2>&1; echo "tail_ab rc=$?"
cat gpurun_out/r02e_tail_ab.json | head -30
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02e_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r02e_bench.log | cut -c1-800
