cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:ktc_verify_partial -c 1 -o gpurun_out/prof_verify python tools/profile_winners.py conv3 > /dev/null 2>&1; echo "ncu rc=$?"
