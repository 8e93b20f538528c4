cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ktc_verify_partial -c 1 -o gpurun_out/prof_verify2 python tools/profile_winners.py conv3 > /dev/null 2>&1; echo "ncu rc=$?"
