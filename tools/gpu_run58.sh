cd $GRAFT_REPO_ROOT
for wl in cfg2 cfg3 cfg5; do
  timeout 600 python bench.py --slab --workload $wl --steps 3 --warmup 3 --no-cpu --no-ttr --secondary "" --no-rank-proxy > gpurun_out/slab_$wl.log 2>&1; echo "$wl rc=$?"; tail -4 gpurun_out/slab_$wl.log | cut -c1-400
done
