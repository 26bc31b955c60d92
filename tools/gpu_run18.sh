cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_var_fused.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/vtb_tests.log 2>&1; echo "vtb tests rc=$?"; tail -5 gpurun_out/vtb_tests.log
VAR_STEPS=40 VAR_FUSE=1,2 VAR_SHAPES=4096x4096,2048x2048,1024x1024 timeout 300 python tools/var_probe.py > gpurun_out/var_probe3.log 2>&1; echo "var rc=$?"; cat gpurun_out/var_probe3.log
