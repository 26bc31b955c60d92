cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SECONDS=0
timeout 900 python bench.py > gpurun_out/bench_v7.log 2> gpurun_out/bench_v7.err; echo "bench rc=$? in ${SECONDS}s"; tail -1 gpurun_out/bench_v7.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['clocks']); print(json.dumps(d['multi_gpu_rank_proxy'], indent=1))"
