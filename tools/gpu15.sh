cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -m gpu -x > gpurun_out/r15_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r15_pytest.log
for v in 0 1; do
  KTC_CONV_F2=$v timeout 900 python tools/compile_ab.py --families conv5,conv7,conv9,conv11 --out gpurun_out/cf2_$v.json 2>&1 | tail -4
done
python tools/compile_ab.py --compare gpurun_out/cf2_0.json gpurun_out/cf2_1.json
