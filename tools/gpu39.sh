cd $GRAFT_REPO_ROOT
export KTC_SEGV_TRACE=1
timeout 1500 python -m pytest tests/test_gpu_ptxgen.py -q -x 2>&1 | tail -6
for v in nvrtc ptx; do
  KTC_GEMM_CODEGEN=$v timeout 900 python tools/gemm_probe.py --size 2048 --out gpurun_out/gp_$v.json 2>&1 | tail -2
  KTC_GEMM_CODEGEN=$v timeout 900 python tools/gemm_probe.py --size 4096 --out gpurun_out/gp4_$v.json 2>&1 | tail -2
done
python tools/gemm_probe.py --compare gpurun_out/gp_nvrtc.json gpurun_out/gp_ptx.json
python tools/gemm_probe.py --compare gpurun_out/gp4_nvrtc.json gpurun_out/gp4_ptx.json
