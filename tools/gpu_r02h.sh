# Launch-overhead probe (per-launch events vs one stream), configs[3] skinny
# shape searches under the split policy, then full-search shard 2:
#   gpurun --timeout 4500 -- 'bash tools/gpu_r02h.sh'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python tools/launch_overhead_probe.py > gpurun_out/r02h_overhead.log 2>&1; echo overhead rc=$?
cat gpurun_out/r02h_overhead.log | cut -c1-300
timeout 900 python tools/gemm_shape_search.py 8192x256x8192 0.0156 > gpurun_out/r02h_skinny1.log 2>&1; echo skinny1 rc=$?
cut -c1-600 gpurun_out/r02h_skinny1.log
timeout 600 python tools/gemm_shape_search.py 4096x4096x256 0.0156 > gpurun_out/r02h_skinny2.log 2>&1; echo skinny2 rc=$?
cut -c1-600 gpurun_out/r02h_skinny2.log
FS_TIMEOUT=${FS_T:-2700} bash tools/gpu_fullsearch_4096.sh 284204 142102
