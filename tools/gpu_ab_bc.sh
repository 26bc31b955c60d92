cd $GRAFT_REPO_ROOT
rm -f gpurun_out/ab_bc.log
for v in "$@"; do SRJ_LIB_PATH=build/ab/$v/libsrj.so timeout 300 python tools/bc_probe.py | grep '"fuse": 4' | sed "s/^/$v /" >> gpurun_out/ab_bc.log; done
cat gpurun_out/ab_bc.log
