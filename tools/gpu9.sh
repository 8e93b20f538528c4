cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r9_smi.txt 2>&1
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/r9_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r9_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r9_smoke.log 2>&1; echo "smoke rc=$?"
tail -2 gpurun_out/r9_smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r9_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r9_bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r9_bench_ref.log 2>&1; echo "ref rc=$?"
tail -1 gpurun_out/r9_bench_ref.log
