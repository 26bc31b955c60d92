cd $GRAFT_REPO_ROOT
CMD="env VAR_STEPS=8 VAR_FUSE=2 VAR_SHAPES=4096x4096 python tools/var_probe.py"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sweep2d_vtb -s 2 -c 1 -o gpurun_out/prof_vtb $CMD > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
