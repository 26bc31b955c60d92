cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_r2_v4.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputests_r2_v4.log
(
timeout 300 python tools/slab_rank_probe.py cfg2 4096 4096 --fuse 4 --steps 2000
timeout 300 python tools/slab_rank_probe.py cfg2 1024 4096 --fuse 4 --steps 4000
timeout 300 python tools/slab_rank_probe.py cfg2 512 4096 --fuse 4 --steps 4000
timeout 300 python tools/slab_rank_probe.py cfg4 16384 32768 --fuse 4 --steps 100
timeout 300 python tools/slab_rank_probe.py cfg4 4096 32768 --fuse 4 --steps 400
timeout 300 python tools/slab_rank_probe.py cfg3 512 512 512 --fuse 2 --steps 200
timeout 300 python tools/slab_rank_probe.py cfg3 256 512 512 --fuse 2 --steps 200
timeout 300 python tools/slab_rank_probe.py cfg3 128 512 512 --fuse 2 --steps 400
timeout 300 python tools/slab_rank_probe.py cfg3 64 512 512 --fuse 2 --steps 800
timeout 300 python tools/slab_rank_probe.py cfg5 32 256 256 --fuse 2 --steps 1600
) > gpurun_out/slab_rank_probe_final.log 2>&1; cut -c1-260 gpurun_out/slab_rank_probe_final.log
