# One shard of the configs[4] full search (4096^3, all 852,608 configurations),
# checkpointed:  gpurun --timeout 3300 -- 'bash tools/gpu_fullsearch_4096.sh <start> <count>'
cd "${GRAFT_REPO_ROOT:-.}"
start=$1; count=$2
ck=profiles/fullsearch_4096/ckpt/ckpt_$(printf %07d $start).csv
export KTC_GEMM_TAIL=0 KTC_GEMM_SK=0  # every shard with the same kernel family as shard 0 (neither switch applies at 4096^3)
timeout ${FS_TIMEOUT:-3200} python tools/gemm_full_search.py --size 4096 --start $start --count $count --prune 2 \
    --dump-times --checkpoint $ck > gpurun_out/fs4096_$(printf %07d $start).log 2>&1
echo "shard $start rc=$?"; tail -1 gpurun_out/fs4096_$(printf %07d $start).log | cut -c1-300
