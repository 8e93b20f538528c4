# Same-box check: full bench vs --no-tuned --no-cpu bench
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r02bb
timeout 600 python bench.py --steps 20 --warmup 5 --no-tuned --no-cpu > gpurun_out/r02bb/b1.log 2>&1
echo "no-tuned: $(tail -1 gpurun_out/r02bb/b1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1))")"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02bb/b2.log 2>&1
echo "full: $(tail -1 gpurun_out/r02bb/b2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1))")"
timeout 600 python bench.py --steps 20 --warmup 5 --no-tuned --no-cpu > gpurun_out/r02bb/b3.log 2>&1
echo "no-tuned: $(tail -1 gpurun_out/r02bb/b3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1))")"
nproc; lscpu | grep "Model name"
