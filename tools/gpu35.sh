cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/b200_winners.json
timeout 3000 python tools/tune_sweep.py --tag r01c --gemm-fraction 0.0078125 --tf32 > gpurun_out/sweep_r01c.log 2>&1; echo "sweep rc=$?"
grep -E "^conv|^gemm" gpurun_out/sweep_r01c.log | cut -c1-200
