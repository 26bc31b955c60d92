cd $GRAFT_REPO_ROOT
C1="python tools/probe3d.py --sizes 512 --workloads cfg3 --steps 24 --reps 1"
C2="python tools/probe3d.py --sizes 256 --workloads cfg5 --steps 24 --reps 1"
$C1 > gpurun_out/plain1.log 2>&1 && $C2 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep3d_rs -s 14 -c 1 -o gpurun_out/prof_rs512_r2 $C1 > gpurun_out/ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep3d_rs -s 14 -c 1 -o gpurun_out/prof_rs256nl_r2 $C2 > gpurun_out/ncu2.log 2>&1; echo "ncu rc=$?"
