cd $GRAFT_REPO_ROOT
timeout 300 /usr/local/cuda/bin/cuda-gdb -batch -ex "set pagination off" -ex run -ex bt -ex "info threads" --args python tools/repro1.py 2>&1 | tail -60
