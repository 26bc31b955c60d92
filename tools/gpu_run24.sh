cd $GRAFT_REPO_ROOT
SRJ_REF_RANDOM_CASES=200 timeout 1500 python -m pytest tests/test_gpu_reference_random.py -q --timeout 1200 -p no:cacheprovider > gpurun_out/refrandom.log 2>&1; echo "rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/refrandom.log | head -20
