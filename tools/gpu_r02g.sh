# TF32 CTA-pair first light + TF32 full search per size, SGEMM split policy per
# tile shape at 2048^3, conv register-budget A/B, then full-search shard 1:
#   gpurun --timeout 4200 -- 'bash tools/gpu_r02g.sh'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 300 python tools/tf32_pair_check.py > gpurun_out/r02g_tf32_pair.log 2>&1; echo pair rc=$?
cat gpurun_out/r02g_tf32_pair.log | cut -c1-300
if grep -q "2048x2048x2048 {'BN': 256, 'BK': 32, 'STAGES': 4, 'CG': 2}: ok pass" gpurun_out/r02g_tf32_pair.log; then
  timeout 900 python tools/tf32_probe.py 2048 4096 8192 > gpurun_out/r02g_tf32_probe.log 2>&1; echo probe rc=$?
  cat gpurun_out/r02g_tf32_probe.log
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_large.py -q -k "tf32 or split_k" 2>&1 | tail -3
fi
timeout 900 python tools/split_probe.py --per-tile 6 --shapes 2048x2048x2048 --splits 0,1,2,3 > gpurun_out/r02g_split.log 2>&1; echo split rc=$?
cut -c1-900 gpurun_out/r02g_split.log
timeout 600 python tools/conv_trace.py > gpurun_out/r02g_conv_trace.log 2>&1; echo trace rc=$?
cut -c1-1500 gpurun_out/r02g_conv_trace.log
timeout 900 python tools/conv_occ_ab.py > gpurun_out/r02g_conv_occ.log 2>&1; echo occ rc=$?
tail -6 gpurun_out/r02g_conv_occ.log | cut -c1-400
FS_TIMEOUT=${FS_T:-2400} bash tools/gpu_fullsearch_4096.sh 142102 142102
