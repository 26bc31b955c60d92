cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_coef_classes.py tests/test_gpu_random.py tests/test_gpu_reference_random.py tests/test_gpu_reference_dropin.py -m gpu -q -x 2>&1 | tail -2
for v in pf1 ptr2; do
  echo "== $v"; SRJ_LIB_PATH=build/ab/$v/libsrj.so timeout 300 python tools/probe.py --fuse "" --three 512,256 --nl 1 2>&1 | grep '"fuse": 1' | cut -c1-120
  SRJ_LIB_PATH=build/ab/$v/libsrj.so timeout 300 python tools/coef_class_probe.py 2>&1 | tail -4 | cut -c1-140
done
