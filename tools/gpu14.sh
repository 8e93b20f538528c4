cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in 0 1; do
  KTC_GEMM_F2=$v timeout 900 python tools/gemm_probe.py --size 2048 --out gpurun_out/probe_f2_$v.json 2>&1 | tail -5
done
python tools/gemm_probe.py --compare gpurun_out/probe_f2_0.json gpurun_out/probe_f2_1.json
for v in 0 1; do
  KTC_GEMM_F2=$v timeout 900 python tools/gemm_probe.py --size 4096 --out gpurun_out/probe4k_f2_$v.json 2>&1 | tail -5
done
python tools/gemm_probe.py --compare gpurun_out/probe4k_f2_0.json gpurun_out/probe4k_f2_1.json
