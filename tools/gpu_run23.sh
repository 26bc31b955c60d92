cd $GRAFT_REPO_ROOT
SRJ_REF_RANDOM_CASES=600 timeout 1500 python -m pytest tests/test_gpu_reference_random.py -q --timeout 1200 -p no:cacheprovider > gpurun_out/refrandom600.log 2>&1; echo "rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/refrandom600.log | head -20
SRJ_RANDOM_CASES=400 timeout 1200 python -m pytest tests/test_gpu_random.py -q --timeout 1000 -p no:cacheprovider > gpurun_out/random400.log 2>&1; echo "rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/random400.log | head -20
