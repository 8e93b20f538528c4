cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export KTC_SEGV_TRACE=1
timeout 1500 python -m pytest tests/test_gpu_ptxgen.py -q -x 2>&1 | tail -15
for v in nvrtc ptx; do
  KTC_CONV_CODEGEN=$v timeout 900 python tools/compile_ab.py --families conv3,conv7,conv11 --out gpurun_out/cg_$v.json 2>&1 | tail -3
done
python tools/compile_ab.py --compare gpurun_out/cg_nvrtc.json gpurun_out/cg_ptx.json
