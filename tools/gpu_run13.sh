cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_reference_dropin.py -q --timeout 800 -p no:cacheprovider > gpurun_out/dropin.log 2>&1; echo "dropin rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/dropin.log | head -30
