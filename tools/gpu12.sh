cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in 0 1; do
  KTC_GEMM_FRAG=$v timeout 900 python tools/gemm_probe.py --size 2048 --out gpurun_out/probe_frag$v.json 2>&1 | tail -9
done
python tools/gemm_probe.py --compare gpurun_out/probe_frag0.json gpurun_out/probe_frag1.json
for v in 0 1; do
  KTC_GEMM_FRAG=$v timeout 900 python tools/gemm_probe.py --size 4096 --out gpurun_out/probe4k_frag$v.json 2>&1 | tail -4
done
python tools/gemm_probe.py --compare gpurun_out/probe4k_frag0.json gpurun_out/probe4k_frag1.json
