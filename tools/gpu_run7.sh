cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_var_fused.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/vtb_tests.log 2>&1; echo "vtb tests rc=$?"; tail -25 gpurun_out/vtb_tests.log
VAR_FUSE=1,2 timeout 300 python tools/var_probe.py > gpurun_out/var_probe.log 2>&1; echo "var rc=$?"; cat gpurun_out/var_probe.log
