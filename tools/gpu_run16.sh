cd $GRAFT_REPO_ROOT
timeout 300 python tools/residual_probe.py > gpurun_out/resid_probe.log 2>&1; echo "probe rc=$?"; cat gpurun_out/resid_probe.log
CMD="env RESID_REPS=1 python tools/residual_probe.py"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:residual -c 12 -o gpurun_out/prof_resid $CMD > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
