# Compile batch-size A/B on the bench's tuning throughput:  gpurun --timeout 1800 -- 'bash tools/gpu_r02z.sh'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r02z
for b in ${BATCHES:-1 8 1 8}; do
  KTC_COMPILE_BATCH=$b timeout 600 python bench.py --steps 20 --warmup 5 --no-tuned --no-cpu > gpurun_out/r02z/bench_b$b.log 2>&1
  echo "batch $b: $(tail -1 gpurun_out/r02z/bench_b$b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1))")"
done
