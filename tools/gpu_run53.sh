cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab_streams.py -m gpu -q -k "slab or emulated or flag_protocol" 2>&1 | tail -8
timeout 300 python tools/slab_rank_probe.py cfg2 4096 4096 --fuse 4 --steps 1000 | cut -c1-200
