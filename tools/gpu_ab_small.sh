cd $GRAFT_REPO_ROOT
# A/B of the small-grid (cluster) path: cfg1 256^2 and the paper's 300^2 per-cell size
rm -f gpurun_out/ab_small.log
for rep in 1 2; do for v in "$@"; do
  SRJ_LIB_PATH=build/ab/$v/libsrj.so timeout 120 python tools/small_probe.py --n 256 --steps 2640 | sed "s/^/$v /" >> gpurun_out/ab_small.log
  SRJ_LIB_PATH=build/ab/$v/libsrj.so VAR_STEPS=400 VAR_FUSE=1 VAR_SHAPES=300x300 timeout 120 python tools/var_probe.py > gpurun_out/vp.tmp 2>&1; sed "s/^/$v /" gpurun_out/vp.tmp >> gpurun_out/ab_small.log
done; done
cat gpurun_out/ab_small.log
