cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_reference_random.py -q --timeout 800 -p no:cacheprovider > gpurun_out/refrandom.log 2>&1; echo "refrandom rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/refrandom.log | head -30
