cd $GRAFT_REPO_ROOT
VAR_STEPS=400 VAR_FUSE=1,2 VAR_SHAPES=300x300,1024x1024,2048x2048 timeout 300 python tools/var_probe.py > gpurun_out/var_probe2.log 2>&1; echo "var rc=$?"; cat gpurun_out/var_probe2.log
