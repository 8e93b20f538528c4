cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "verifier" > gpurun_out/r23_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r23_pytest.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/r23_verify.csv -k regex:ktc_verify python tools/profile_winners.py conv3 conv11 gemm > /dev/null 2>&1; echo "ncu rc=$?"
grep -E "verify" gpurun_out/r23_verify.csv | cut -d, -f5,12- | head -12
