cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/solve_times.py > gpurun_out/solve_times_r2.log 2>&1; echo rc=$?; cut -c1-330 gpurun_out/solve_times_r2.log
timeout 600 python tools/paper_gs.py > gpurun_out/paper_gs_r2.log 2>&1; echo rc=$?; tail -8 gpurun_out/paper_gs_r2.log | cut -c1-300
