cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_reference_dropin.py -q -x --timeout 500 -p no:cacheprovider > gpurun_out/dropin.log 2>&1; echo "dropin rc=$?"; tail -30 gpurun_out/dropin.log
timeout 300 python tools/slab_overhead.py 8 > gpurun_out/slab_overhead.log 2>&1; echo "slab rc=$?"; tail -1 gpurun_out/slab_overhead.log
