# compute-sanitizer over every kernel family (run under gpurun from the repo root):
#   gpurun --timeout 2400 -- 'bash tools/gpu_sanitize.sh'
# Logs: gpurun_out/sanitizer/<tool>.log (summaries copied to profiles/sanitizer_r02/).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/sanitizer
CS=/usr/local/cuda/bin/compute-sanitizer
# the compile pool's threads are host-only; one timed launch per configuration
export KTC_COMPILE_THREADS=8
for tool in memcheck synccheck racecheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check no --report-api-errors no"
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  timeout 900 $CS --tool $tool $extra --print-limit 50 python tools/sanitize_configs.py \
      > gpurun_out/sanitizer/$tool.log 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/sanitizer/$tool.log
done
# negative control: memcheck must flag the out-of-bounds write of a custom kernel
timeout 600 $CS --tool memcheck --leak-check no --print-limit 5 python tools/sanitize_configs.py --control \
    > gpurun_out/sanitizer/memcheck_control.log 2>&1
echo "memcheck control rc=$? (expect errors reported)"; grep -m3 "Invalid\|ERROR SUMMARY" gpurun_out/sanitizer/memcheck_control.log
