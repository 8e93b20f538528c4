# Round-2 pass b: fault tests, fresh-job timeline, sanitizers, ncu of the
# winners not captured in round 1.   gpurun --timeout 3000 -- 'bash tools/gpu_r02b.sh'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r02b
timeout 600 python -m pytest tests/test_gpu_faults.py -q > gpurun_out/r02b/faults.log 2>&1; echo "faults rc=$?"; tail -3 gpurun_out/r02b/faults.log
KTC_TRACE=1 timeout 300 python tools/e2e_probe.py --chunk 25 --jobs 4 > gpurun_out/r02b/e2e_probe.log 2>&1; echo "e2e probe rc=$?"
grep -v "^ktc-trace" gpurun_out/r02b/e2e_probe.log | tail -8
bash tools/gpu_sanitize.sh
export KTC_LINEINFO=1
W4096="gemm:4096:$(python -c "import json;print(json.load(open('tuned/b200_winners.json'))['gemm']['4096']['config'])")"
W8192="gemm:8192:$(python -c "import json;print(json.load(open('tuned/b200_winners.json'))['gemm']['8192']['config'])")"
T2048="tf32:2048:$(python -c "import json;print(json.load(open('tuned/b200_winners.json'))['gemm_tf32']['2048']['config'])")"
T8192="tf32:8192:$(python -c "import json;print(json.load(open('tuned/b200_winners.json'))['gemm_tf32']['8192']['config'])")"
i=0
for w in conv7 conv9 "$W4096" "$W8192" "$T2048" "$T8192"; do
  i=$((i+1))
  k=conv2d_k; case "$w" in gemm*) k=gemm_k;; tf32*) k=gemm_tf32_k;; esac
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
      -o gpurun_out/r02b/prof_$i python tools/profile_winners.py "$w" > gpurun_out/r02b/prof_$i.log 2>&1
  echo "prof $i ($w) rc=$?"
done
