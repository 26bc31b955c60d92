cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputests.log
for w in cfg5 cfg3; do timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu --no-ttr --secondary= > gpurun_out/bench_$w.log 2>&1; echo "$w rc=$?"; tail -1 gpurun_out/bench_$w.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'], d['clocks'])"; done
