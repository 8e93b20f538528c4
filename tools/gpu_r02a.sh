# Round-2 validation pass on one B200 (run under gpurun from the repo root):
#   gpurun --timeout 2400 -- 'bash tools/gpu_r02a.sh'
# pytest -m gpu (incl. the large-shape parity), smoke, the driver's bench
# line (N=1, K=20/W=5), --gpus 2 in one process and under torchrun (both GPU
# workers on cuda:0 here), and the reference arm.  Logs in gpurun_out/r02a_*.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
export KTC_SEGV_TRACE=1
nproc > gpurun_out/r02a_nproc.txt
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/r02a_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r02a_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02a_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r02a_bench.log | cut -c1-600
timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-tuned --no-cpu > gpurun_out/r02a_bench_g2.log 2>&1; echo "bench g2 rc=$?"
tail -1 gpurun_out/r02a_bench_g2.log | cut -c1-400
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-tuned > gpurun_out/r02a_bench_tr2.log 2>&1; echo "bench torchrun2 rc=$?"
tail -1 gpurun_out/r02a_bench_tr2.log | cut -c1-400
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02a_ref.log 2>&1; echo "ref rc=$?"
tail -1 gpurun_out/r02a_ref.log | cut -c1-400
