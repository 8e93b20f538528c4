cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export KTC_LINEINFO=1
timeout 600 ncu --set full --clock-control none -k regex:gemm_tf32_k -c 1 -o gpurun_out/prof_tf32_s2 python tools/profile_winners.py "tf32:4096:BK=32;BN=256;STAGES=2" > /dev/null 2>&1; echo "rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:gemm_tf32_k -c 1 -o gpurun_out/prof_tf32_s4 python tools/profile_winners.py "tf32:4096:BK=32;BN=256;STAGES=4" > /dev/null 2>&1; echo "rc=$?"
