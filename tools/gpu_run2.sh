cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/gputests.log
timeout 300 python tools/slab_overhead.py 8 > gpurun_out/slab_overhead.log 2>&1; echo "slab rc=$?"; tail -5 gpurun_out/slab_overhead.log
timeout 600 python bench.py --workload cfg3 --steps 3 --warmup 3 > gpurun_out/bench_cfg3.log 2>&1; echo "cfg3 rc=$?"; tail -c 1500 gpurun_out/bench_cfg3.log
timeout 600 python bench.py --workload cfg5 --steps 3 --warmup 3 > gpurun_out/bench_cfg5.log 2>&1; echo "cfg5 rc=$?"; tail -c 1500 gpurun_out/bench_cfg5.log
