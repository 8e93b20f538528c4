# SA / PSO replicas at BASELINE sizes through the command line (run under gpurun):
#   /usr/local/graft/bin/gpurun --timeout 1800 -- 'bash tools/gpu_replicas.sh'
# `ktune-b200 stats` on the box's one GPU (replicas run one after another;
# --gpus N on an N-GPU node runs N at a time -- sharing one GPU between two
# replica workers would perturb the timings); reports in gpurun_out/replicas/.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/replicas
B=paper_1703_06503_b200/ktune-b200
run() {  # job runs
  local t0=$SECONDS
  timeout 900 $B stats tools/jobs/$1.json --runs $2 --gpus 1 --out gpurun_out/replicas/$1.csv \
      > gpurun_out/replicas/$1.log 2>&1
  echo "$1 rc=$? wall $((SECONDS - t0)) s" | tee -a gpurun_out/replicas/$1.log
  tail -5 gpurun_out/replicas/$1.log
}
run gemm4096_pso6 8
run gemm4096_sa4 8
run gemm8192_pso6 4
