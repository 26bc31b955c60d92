cd $GRAFT_REPO_ROOT
for i in 1 2; do timeout 300 python tools/solve_times.py --configs cfg1 2>&1 | cut -c1-250; done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_dropin.py -m gpu -q -x -k "stopping or solve or divergence or reference" 2>&1 | tail -2
