cd $GRAFT_REPO_ROOT
timeout 300 python tools/probe3d.py > gpurun_out/probe3d_rs.log 2>&1; echo "rs rc=$?"; cat gpurun_out/probe3d_rs.log | tail -4
CMD="python tools/probe3d.py --sizes 512 --workloads cfg3 --steps 24 --reps 1"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sweep3d_rs -s 14 -c 1 -o gpurun_out/prof_rs512c $CMD > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
