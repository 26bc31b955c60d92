cd $GRAFT_REPO_ROOT
# A/B timing of libsrj builds under build/ab/*/ on the per-cell paths
# (coef_class_probe + var_probe); args: variant names
for rep in 1 2; do for v in "$@"; do
  SRJ_LIB_PATH=build/ab/$v/libsrj.so timeout 300 python tools/coef_class_probe.py ${CLS_ARGS} | sed "s/^/$v /" >> gpurun_out/ab_var.log
  SRJ_LIB_PATH=build/ab/$v/libsrj.so VAR_SHAPES=${VAR_SHAPES:-512x512x512} VAR_FUSE=${VAR_FUSE:-1} timeout 300 python tools/var_probe.py | sed "s/^/$v /" >> gpurun_out/ab_var.log
done; done
