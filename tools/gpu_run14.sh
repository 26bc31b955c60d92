cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputests.log
timeout 300 python tools/probe.py --n 4096 --fuse 2,3,4,5,6,8 --three "" --nl 0 --steps 2000 > gpurun_out/probe2d.log 2>&1; cat gpurun_out/probe2d.log
timeout 300 python tools/probe.py --n 32768 --fuse 4 --three "" --nl 0 --steps 64 >> gpurun_out/probe2d.log 2>&1; tail -1 gpurun_out/probe2d.log
