# Round-2 validation of HEAD: full GPU suite, smoke, TF32 search (grouped
# raster), skinny SGEMM search under stream-K, ncu of the new 4096^3 winner,
# the bench line + reference arm, and the bench's ncu launch list.
#   gpurun --timeout 4800 -- 'bash tools/gpu_r02l.sh'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r02l
export KTC_SEGV_TRACE=1
timeout 1800 python -m pytest tests/ -q -m gpu > gpurun_out/r02l/pytest.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/r02l/pytest.log | cut -c1-400
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python tools/tf32_probe.py 2048 4096 8192 > gpurun_out/r02l/tf32_probe.log 2>&1; echo "tf32 rc=$?"; cat gpurun_out/r02l/tf32_probe.log
timeout 900 python tools/gemm_shape_search.py 8192x256x8192 0.0156 > gpurun_out/r02l/skinny1.log 2>&1; echo "skinny rc=$?"; cut -c1-500 gpurun_out/r02l/skinny1.log
W4096="gemm:4096:$(python -c "import json;print(json.load(open('tuned/b200_winners.json'))['gemm']['4096']['config'])")"
KTC_LINEINFO=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_k -c 1 \
    -o gpurun_out/r02l/prof_sgemm4096 python tools/profile_winners.py "$W4096" > gpurun_out/r02l/prof_sgemm4096.log 2>&1; echo "ncu 4096 rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02l/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r02l/bench.log | cut -c1-1500
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02l/bench_ref.log 2>&1; echo "ref rc=$?"
tail -1 gpurun_out/r02l/bench_ref.log | cut -c1-600
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/r02l/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r02l/bench_ncu.log 2>&1; echo "ncu launches rc=$?"
