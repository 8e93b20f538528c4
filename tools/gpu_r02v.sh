# ncu of the configs[3] skinny SGEMM winners:  gpurun --timeout 900 -- 'bash tools/gpu_r02v.sh'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r02v
export KTC_LINEINFO=1
for s in 8192x256x8192 4096x4096x256; do
  w="gemm:$s:$(python -c "import json;print(json.load(open('tuned/b200_winners.json'))['gemm']['$s']['config'])")"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_k -c 1 \
      -o gpurun_out/r02v/prof_$s python tools/profile_winners.py "$w" > gpurun_out/r02v/prof_$s.log 2>&1
  echo "ncu $s rc=$?"; tail -1 gpurun_out/r02v/prof_$s.log
done
