cd $GRAFT_REPO_ROOT
CMD="python tools/probe3d.py --sizes 512 --workloads cfg3 --steps 24 --reps 1"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sweep3d_rs -s 14 -c 2 -o gpurun_out/prof_rs512 $CMD > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu.log
