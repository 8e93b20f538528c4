# Final round-2 validation of HEAD (run under gpurun):
#   gpurun --timeout 3600 -- 'bash tools/gpu_r02o.sh'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r02o
export KTC_SEGV_TRACE=1
timeout 1800 python -m pytest tests/ -q -m gpu > gpurun_out/r02o/pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02o/pytest.log | cut -c1-300
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r02o/bench_default.log 2>&1; echo "bench default rc=$?"
tail -1 gpurun_out/r02o/bench_default.log | cut -c1-400
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02o/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r02o/bench.log | cut -c1-400
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02o/bench_ref.log 2>&1; echo "ref rc=$?"
tail -1 gpurun_out/r02o/bench_ref.log | cut -c1-300
timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-tuned --no-cpu > gpurun_out/r02o/bench_g2.log 2>&1; echo "bench g2 rc=$?"
tail -1 gpurun_out/r02o/bench_g2.log | cut -c1-300
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-tuned > gpurun_out/r02o/bench_tr2.log 2>&1; echo "bench torchrun2 rc=$?"
tail -1 gpurun_out/r02o/bench_tr2.log | cut -c1-300
