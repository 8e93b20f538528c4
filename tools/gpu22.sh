cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
KTC_TRACE=1 timeout 600 python tools/e2e_probe.py > gpurun_out/e2e_probe_trace.log 2>&1; echo "e2e rc=$?"; cat gpurun_out/e2e_probe_trace.log
