cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_r2_v6.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputests_r2_v6.log
