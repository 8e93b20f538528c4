# Split-K launch policy check, conv image-size probe, then the first shard of
# the configs[4] full search:  gpurun --timeout 3900 -- 'bash tools/gpu_r02f.sh'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k split_k 2>&1 | tail -2
timeout 600 python tools/split_probe.py --top 30 --shapes 8192x256x8192,4096x4096x256 --splits 0,1,2 > gpurun_out/r02f_split.log 2>&1; echo split rc=$?
cut -c1-700 gpurun_out/r02f_split.log
timeout 600 python tools/conv_size_probe.py > gpurun_out/r02f_conv_size.log 2>&1; echo conv_size rc=$?
cat gpurun_out/r02f_conv_size.log | cut -c1-200
FS_TIMEOUT=2600 bash tools/gpu_fullsearch_4096.sh 0 142102
