cd $GRAFT_REPO_ROOT
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_default.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['clocks'], d['roofline']['frac'], [ (o['value'], o['clocks']['sm_mhz']) for o in d.get('other_workloads',[])])"
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-ttr --e2e-steps 0 --secondary="
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sweep2d_tb -s 3 -c 1 -o gpurun_out/prof_2d_r2 $CMD > gpurun_out/ncu1.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2.csv $CMD > gpurun_out/ncu2.log 2>&1; echo "ncu rc=$?"
