# Prefetch-window change: bench value on one box (default vs the old 8-deep window)
#   gpurun --timeout 1800 -- 'bash tools/gpu_r02aa.sh'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r02aa
for i in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-tuned --no-cpu > gpurun_out/r02aa/bench_$i.log 2>&1
  echo "default run $i: $(tail -1 gpurun_out/r02aa/bench_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1), round(d['value_warm_cache'],1))")"
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ptxgen.py tests/test_cli.py -q > gpurun_out/r02aa/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02aa/pytest.log | cut -c1-200
