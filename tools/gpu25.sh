cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "verifier" 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/r25_verify.csv -k regex:ktc_verify_partial python tools/profile_winners.py conv3 conv11 gemm > /dev/null 2>&1; echo "ncu rc=$?"
grep -E "verify" gpurun_out/r25_verify.csv | cut -d, -f12- | head -6
