cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_r2_v3.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputests_r2_v3.log
timeout 900 python bench.py > gpurun_out/bench_v6.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_v6.log | cut -c1-600
