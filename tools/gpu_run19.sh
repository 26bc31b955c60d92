cd $GRAFT_REPO_ROOT
free -g | head -2
timeout 900 python bench.py --workload cfg4 --steps 3 --warmup 3 --no-cpu --no-ttr --e2e-steps 0 --secondary= > gpurun_out/bench_cfg4.log 2>&1; echo "cfg4 rc=$?"; tail -2 gpurun_out/bench_cfg4.log | cut -c1-1500
timeout 600 python bench.py --workload cfg1 --steps 20 --warmup 3 --secondary= > gpurun_out/bench_cfg1.log 2>&1; echo "cfg1 rc=$?"; tail -1 gpurun_out/bench_cfg1.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d.get('time_to_residual'), d['cpu_baseline']['value'])"
