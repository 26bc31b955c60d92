cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab_streams.py -m gpu -q -k "slab or emulated or flag_protocol" 2>&1 | tail -3
rm -f gpurun_out/ab2d.log
bash tools/gpu_ab2d.sh before after > /dev/null 2>&1
cat gpurun_out/ab2d.log | cut -c1-100
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
) 2>&1 | tee gpurun_out/slab_rank_probe4.log
