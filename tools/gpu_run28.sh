cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tests/slab_streams_worker.py > gpurun_out/slab_streams.log 2>&1; echo "worker rc=$?"; tail -20 gpurun_out/slab_streams.log
nvidia-smi --query-gpu=name,memory.used --format=csv
