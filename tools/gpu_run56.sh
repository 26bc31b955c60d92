cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random.py -m gpu -q -x -k "small or cluster or random or golden or reference" 2>&1 | tail -2
for rep in 1 2; do for v in base fsm; do
  for n in 64 128 256; do SRJ_LIB_PATH=build/ab/$v/libsrj.so timeout 120 python tools/small_probe.py --n $n --steps 2640 | sed "s/^/$v n=$n /"; done
  SRJ_LIB_PATH=build/ab/$v/libsrj.so VAR_STEPS=400 VAR_FUSE=1 VAR_SHAPES=160x160,300x300 timeout 120 python tools/var_probe.py 2>&1 | sed "s/^/$v /"
done; done
