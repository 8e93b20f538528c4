# Final validation of HEAD + ncu of the TF32 winners (TMA-store epilogue):
#   gpurun --timeout 3000 -- 'bash tools/gpu_r02u.sh'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r02u
export KTC_SEGV_TRACE=1
timeout 1800 python -m pytest tests/ -q -m gpu > gpurun_out/r02u/pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r02u/pytest.log | cut -c1-300
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02u/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r02u/bench.log | cut -c1-300
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02u/bench_ref.log 2>&1; echo "ref rc=$?"
tail -1 gpurun_out/r02u/bench_ref.log | cut -c1-200
export KTC_LINEINFO=1
i=0
for s in 2048 8192; do
  i=$((i+1))
  w="tf32:$s:$(python -c "import json;print(json.load(open('tuned/b200_winners.json'))['gemm_tf32']['$s']['config'])")"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tf32_k -c 1 \
      -o gpurun_out/r02u/prof_tf32_$s python tools/profile_winners.py "$w" > gpurun_out/r02u/prof_tf32_$s.log 2>&1
  echo "ncu tf32 $s rc=$?"
done
