cd $GRAFT_REPO_ROOT
timeout 300 python tools/bc_probe.py > gpurun_out/probe_bc.log 2>&1; cat gpurun_out/probe_bc.log
