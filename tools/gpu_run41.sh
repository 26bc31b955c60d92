cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_slab_streams.py -m gpu -q 2>&1 | tail -3
SRJ_SLAB_FLAG_KERNEL=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "slab or emulated" 2>&1 | tail -2
SRJ_SLAB_FLAG_KERNEL=1 timeout 300 python tools/slab_rank_probe.py cfg3 64 512 512 --fuse 2 --steps 800 | cut -c1-200
