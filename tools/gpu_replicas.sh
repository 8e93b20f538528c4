# SA / PSO replicas at BASELINE sizes through the command line (run under gpurun):
#   /usr/local/graft/bin/gpurun --timeout 1800 -- 'bash tools/gpu_replicas.sh'
# `ktune-b200 stats` on the box's one GPU (replicas run one after another;
# --gpus N on an N-GPU node runs N at a time -- sharing one GPU between two
# replica workers would perturb the timings); reports in gpurun_out/replicas/.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/replicas
B=paper_1703_06503_b200/ktune-b200
for j in gemm4096_pso6 gemm4096_sa4; do
  /usr/bin/time -f "$j wall %e s" timeout 900 $B stats tools/jobs/$j.json --runs 8 --gpus 1 \
      --out gpurun_out/replicas/$j.csv > gpurun_out/replicas/$j.log 2>&1; echo "$j rc=$?"
  cat gpurun_out/replicas/$j.log | tail -4
done
/usr/bin/time -f "gemm8192_pso6 wall %e s" timeout 900 $B stats tools/jobs/gemm8192_pso6.json --runs 4 \
    --gpus 1 --out gpurun_out/replicas/gemm8192_pso6.csv > gpurun_out/replicas/gemm8192_pso6.log 2>&1
echo "gemm8192_pso6 rc=$?"; tail -4 gpurun_out/replicas/gemm8192_pso6.log
