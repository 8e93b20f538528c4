# Compile ordering A/B (longest-first vs FIFO) on one box
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r02cc
for o in lpt fifo lpt fifo; do
  KTC_COMPILE_ORDER=$o timeout 600 python bench.py --steps 20 --warmup 5 --no-tuned --no-cpu > gpurun_out/r02cc/b_$o.log 2>&1
  echo "$o: $(tail -1 gpurun_out/r02cc/b_$o.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1))")"
done
