cd $GRAFT_REPO_ROOT
# A/B timing of libsrj builds (build/ab/<name>/) on the 2D cfg2 kernel
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv -lms 500 > gpurun_out/ab_clocks.csv &
SMI=$!
for rep in 1 2 3; do for v in "$@"; do
  SRJ_LIB_PATH=build/ab/$v/libsrj.so timeout 300 python tools/probe.py --n 4096 --fuse 4 --three "" --nl 0 --steps 2000 | sed "s/^/$v /" >> gpurun_out/ab2d.log
done; done
kill $SMI
cat gpurun_out/ab2d.log
