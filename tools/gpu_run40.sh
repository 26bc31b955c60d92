cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab_streams.py -m gpu -q -k "slab or emulated or flag_protocol" 2>&1 | tail -3
SRJ_SLAB_DIRECT=0 timeout 300 python tests/slab_streams_worker.py 2>&1 | tail -1
(
timeout 300 python tools/slab_rank_probe.py cfg2 4096 4096 --fuse 4 --steps 2000
timeout 300 python tools/slab_rank_probe.py cfg2 1024 4096 --fuse 4 --steps 4000
timeout 300 python tools/slab_rank_probe.py cfg2 512 4096 --fuse 4 --steps 4000
timeout 300 python tools/slab_rank_probe.py cfg4 4096 32768 --fuse 4 --steps 400
timeout 300 python tools/slab_rank_probe.py cfg3 512 512 512 --fuse 2 --steps 200
timeout 300 python tools/slab_rank_probe.py cfg3 256 512 512 --fuse 2 --steps 200
timeout 300 python tools/slab_rank_probe.py cfg3 128 512 512 --fuse 2 --steps 400
timeout 300 python tools/slab_rank_probe.py cfg3 64 512 512 --fuse 2 --steps 800
timeout 300 python tools/slab_rank_probe.py cfg5 32 256 256 --fuse 2 --steps 1600
) > gpurun_out/slab_rank_probe_final2.log 2>&1; cut -c1-175 gpurun_out/slab_rank_probe_final2.log
