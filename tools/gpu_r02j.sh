# ncu of the new winners (TF32 CTA pairs, split-K skinny SGEMM), TF32/split
# GPU tests, then full-search shard 4:  gpurun --timeout 4500 -- 'bash tools/gpu_r02j.sh'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r02j
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_large.py -q -k "tf32 or split_k" > gpurun_out/r02j/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02j/pytest.log
export KTC_LINEINFO=1
T2048="tf32:2048:$(python -c "import json;print(json.load(open('tuned/b200_winners.json'))['gemm_tf32']['2048']['config'])")"
T8192="tf32:8192:$(python -c "import json;print(json.load(open('tuned/b200_winners.json'))['gemm_tf32']['8192']['config'])")"
S1="gemm:8192x256x8192:$(python -c "import json;print(json.load(open('tuned/b200_winners.json'))['gemm']['8192x256x8192']['config'])")"
i=0
for w in "$T2048" "$T8192" "$S1"; do
  i=$((i+1))
  k=gemm_k; case "$w" in tf32*) k=gemm_tf32_k;; esac
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
      -o gpurun_out/r02j/prof_$i python tools/profile_winners.py "$w" > gpurun_out/r02j/prof_$i.log 2>&1
  echo "prof $i ($w) rc=$?"
done
unset KTC_LINEINFO
FS_TIMEOUT=${FS_T:-2800} bash tools/gpu_fullsearch_4096.sh 568408 142102
