cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in 0 1; do KTC_CONV_OSTREAM=$v timeout 600 python tools/conv_sustained_ab.py --filters 3,5,7 --out gpurun_out/os$v.json 2>&1 | tail -3; done
python tools/conv_sustained_ab.py --compare gpurun_out/os0.json gpurun_out/os1.json
