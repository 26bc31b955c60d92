cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_bench_launcher.py -m gpu -q 2>&1 | tail -3
