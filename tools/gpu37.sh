cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01c
export KTC_LINEINFO=1
for w in conv3 conv5 conv7 conv11 gemm; do
  k=conv2d_k; [ $w = gemm ] && k=gemm_k
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/r01c/prof_$w python tools/profile_winners.py $w > gpurun_out/r01c/prof_$w.log 2>&1
  echo "$w rc=$?"
done
unset KTC_LINEINFO
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01c/launches_bench.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r01c/launches_bench.log 2>&1; echo "launch list rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r37_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r37_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['clocks'])"
