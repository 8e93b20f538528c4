cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export KTC_SEGV_TRACE=1
timeout 600 python tools/tf32_repro.py 2 > gpurun_out/tf32_repro.log 2>&1; echo "repro rc=$?"
tail -45 gpurun_out/tf32_repro.log
timeout 600 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1; echo "e2e rc=$?"; cat gpurun_out/e2e_probe.log
