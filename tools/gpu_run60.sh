cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random.py tests/test_gpu_reference_random.py -m gpu -q -x 2>&1 | tail -2
for mp in 8 4 2 1; do
  echo "== min planes $mp"
  for n in 32 64 96 128 192; do
    SRJ_MIN_PLANES=$mp timeout 120 python tools/probe3d.py --sizes $n --workloads cfg3 --steps 400 --reps 2 2>&1 | cut -c1-130
  done
done
