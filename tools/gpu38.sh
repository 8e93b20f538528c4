cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_ptxgen.py -q -x 2>&1 | tail -3
for v in nvrtc ptx; do
  KTC_CONV_CODEGEN=$v timeout 900 python tools/compile_ab.py --families conv3,conv5,conv7 --out gpurun_out/cg2_$v.json 2>&1 | tail -3
done
python tools/compile_ab.py --compare gpurun_out/cg2_nvrtc.json gpurun_out/cg2_ptx.json
