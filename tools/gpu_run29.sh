cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tests/slab_streams_worker.py > gpurun_out/slab_streams2.log 2>&1; echo "worker rc=$?"; tail -4 gpurun_out/slab_streams2.log
SRJ_SLAB_SPLIT=0 timeout 300 python tests/slab_streams_worker.py > gpurun_out/slab_streams2_nosplit.log 2>&1; echo "worker(nosplit) rc=$?"; tail -2 gpurun_out/slab_streams2_nosplit.log
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "slab or emulated" 2>&1 | tail -3
(
timeout 300 python tools/slab_rank_probe.py cfg2 4096 4096 --fuse 4 --steps 2000
timeout 300 python tools/slab_rank_probe.py cfg2 1024 4096 --fuse 4 --steps 4000
timeout 300 python tools/slab_rank_probe.py cfg4 4096 32768 --fuse 4 --steps 400
timeout 300 python tools/slab_rank_probe.py cfg3 512 512 512 --fuse 2 --steps 200
timeout 300 python tools/slab_rank_probe.py cfg3 128 512 512 --fuse 2 --steps 400
timeout 300 python tools/slab_rank_probe.py cfg3 64 512 512 --fuse 2 --steps 800
timeout 300 python tools/slab_rank_probe.py cfg5 32 256 256 --fuse 2 --steps 1600
) > gpurun_out/slab_rank_probe.log 2>&1; cat gpurun_out/slab_rank_probe.log
