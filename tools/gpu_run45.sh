cd $GRAFT_REPO_ROOT
timeout 300 python tools/call_overhead.py
