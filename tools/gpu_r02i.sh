# conv persistent-CTA A/B (verified), then full-search shard 3:
#   gpurun --timeout 4500 -- 'bash tools/gpu_r02i.sh'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python tools/conv_occ_ab.py --variants "base:;persist:KTC_CONV_PERSIST=1;persist16:KTC_CONV_PERSIST=1,KTC_CONV_MINCTA=16;persistsm:KTC_CONV_PERSIST=1,KTC_CONV_MINCTA=1" > gpurun_out/r02i_persist.log 2>&1; echo persist rc=$?
tail -8 gpurun_out/r02i_persist.log | cut -c1-700
FS_TIMEOUT=${FS_T:-2700} bash tools/gpu_fullsearch_4096.sh 426306 142102
