cd $GRAFT_REPO_ROOT
timeout 300 python tools/call_overhead.py 2>&1 | head -12
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_r2_v5.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputests_r2_v5.log
