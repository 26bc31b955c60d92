cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/probe.py --fuse "" --three 512 --nl 0 > gpurun_out/plain_t1.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sweep3d -s 6 -c 2 -o gpurun_out/prof_3d_t1 python tools/probe.py --fuse "" --three 512 --nl 0 > gpurun_out/ncu_t1.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_t1.log
ls -la gpurun_out/*.ncu-rep
