cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 3000 python tools/gemm_sweeps.py --sample 2048 > gpurun_out/gemm_sweeps_r01b.log 2>&1; echo "sweeps rc=$?"
cut -c1-250 gpurun_out/gemm_sweeps_r01b.log | tail -16
