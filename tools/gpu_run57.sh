cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_r2_v7.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputests_r2_v7.log
timeout 900 python bench.py > gpurun_out/bench_v9.log 2> gpurun_out/bench_v9.err; echo "bench rc=$?"; tail -1 gpurun_out/bench_v9.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['clocks'], d['roofline']['frac'], d['time_to_residual']['seconds'], [(o['value'], o['clocks']['sm_mhz']) for o in d['other_workloads']], [c['rank_efficiency'] for c in d['multi_gpu_rank_proxy']['cases']])"
