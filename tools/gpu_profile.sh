# ncu evidence for the tuned winners (tuned/b200_winners.json) and the bench
# command's launch list (run under gpurun; copy summaries into profiles/<round>/):
#   /usr/local/graft/bin/gpurun --timeout 1800 -- 'bash tools/gpu_profile.sh r02'
cd "${GRAFT_REPO_ROOT:-.}"
tag=${1:-scratch}
mkdir -p gpurun_out/$tag
export KTC_LINEINFO=1
for w in conv3 conv5 conv7 conv11 gemm; do
  k=conv2d_k; [ $w = gemm ] && k=gemm_k
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
      -o gpurun_out/$tag/prof_$w python tools/profile_winners.py $w > gpurun_out/$tag/prof_$w.log 2>&1
  echo "$w rc=$?"
done
unset KTC_LINEINFO
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/$tag/launches_bench.csv python bench.py --steps 2 --warmup 3 \
    > gpurun_out/$tag/launches_bench.log 2>&1
echo "launch list rc=$?"
