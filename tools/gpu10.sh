cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for m in 0 min mid; do
  KTC_FAST_COMPILE=$m timeout 900 python tools/compile_ab.py --out gpurun_out/cab_$m.json 2>&1 | tail -4
done
python tools/compile_ab.py --compare gpurun_out/cab_0.json gpurun_out/cab_min.json
python tools/compile_ab.py --compare gpurun_out/cab_0.json gpurun_out/cab_mid.json
KTC_FAST_COMPILE=min timeout 900 python bench.py --steps 5 --warmup 3 --no-tuned > gpurun_out/r10_bench_min.log 2>&1; tail -1 gpurun_out/r10_bench_min.log | cut -c1-300
