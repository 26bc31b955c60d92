cd $GRAFT_REPO_ROOT
timeout 600 python tools/self_slab_probe.py 4096
