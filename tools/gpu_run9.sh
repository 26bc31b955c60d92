cd $GRAFT_REPO_ROOT
timeout 300 python tools/slab_overhead.py 8 > gpurun_out/slab_overhead.log 2>&1; echo "slab rc=$?"; tail -2 gpurun_out/slab_overhead.log
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider -k "slab or ipc or distributed or Slab" > gpurun_out/slab_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/slab_tests.log
