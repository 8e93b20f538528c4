# Tuning sweeps (run under gpurun): full conv searches per filter, SGEMM random
# search at 2048^3, TF32 variant, then configs[3]/[4] (shape sweep, 4096 sample).
#   /usr/local/graft/bin/gpurun --timeout 3300 -- 'bash tools/gpu_sweeps.sh r02'
cd "${GRAFT_REPO_ROOT:-.}"
tag=${1:-scratch}
mkdir -p gpurun_out
timeout 2400 python tools/tune_sweep.py --tag $tag --gemm-fraction 0.03125 --tf32 \
    > gpurun_out/sweep_$tag.log 2>&1; echo "sweep rc=$?"
timeout 3000 python tools/gemm_sweeps.py --sample 2048 --prune 2.0 \
    > gpurun_out/gemm_sweeps_$tag.log 2>&1; echo "gemm sweeps rc=$?"
