cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_line.py tests/test_gpu_reference_dropin.py -m gpu -x -q > gpurun_out/line_tests.log 2>&1; echo "line rc=$?"; tail -30 gpurun_out/line_tests.log
timeout 900 python -m pytest tests/test_gpu_reference_random.py -m gpu -q -k "60 or 61 or 62 or 63 or 64 or 65 or 66 or 67 or 68 or 69 or 70 or 71" > gpurun_out/line_random.log 2>&1; echo "rand rc=$?"; tail -15 gpurun_out/line_random.log
