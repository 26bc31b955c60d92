cd $GRAFT_REPO_ROOT
SRJ_RS3D=0 timeout 300 python tools/probe3d.py > gpurun_out/probe3d_tb.log 2>&1; echo "tb rc=$?"; cat gpurun_out/probe3d_tb.log | tail -4
timeout 300 python tools/probe3d.py > gpurun_out/probe3d_rs.log 2>&1; echo "rs rc=$?"; cat gpurun_out/probe3d_rs.log | tail -4
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/gputests.log
