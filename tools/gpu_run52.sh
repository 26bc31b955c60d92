cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab_streams.py -m gpu -q -k "slab or emulated or flag_protocol" 2>&1 | tail -8
