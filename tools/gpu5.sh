cd $GRAFT_REPO_ROOT
timeout 300 python tools/tf32_debug.py 2>&1 | tail -30
KTC_TF32_DESC_VARIANT=1 timeout 300 python tools/tf32_debug.py 2>&1 | tail -12
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python tools/profile_winners.py conv3 conv11 gemm > gpurun_out/launches_r01.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv2d_k -c 1 -o gpurun_out/prof_conv3_r01 python tools/profile_winners.py conv3 > gpurun_out/prof_conv3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv2d_k -c 1 -o gpurun_out/prof_conv11_r01 python tools/profile_winners.py conv11 > gpurun_out/prof_conv11.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_k -c 1 -o gpurun_out/prof_gemm_r01 python tools/profile_winners.py gemm > gpurun_out/prof_gemm.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 2>&1 | tail -3
ls -la gpurun_out
