cd $GRAFT_REPO_ROOT
VAR_FUSE=1,2,3,4 timeout 300 python tools/var_probe.py > gpurun_out/var_probe.log 2>&1; echo "var rc=$?"; cat gpurun_out/var_probe.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_cfg2.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_cfg2.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['clocks']); [print(o['workload'][:20], o['value'], o['clocks']) for o in d.get('other_workloads',[])]"
