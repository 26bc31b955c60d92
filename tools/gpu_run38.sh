cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "dense_kernel" 2>&1 | tail -2
for v in after j3 j4; do
  echo "== $v"; SRJ_LIB_PATH=build/ab/$v/libsrj.so timeout 300 python tools/probe.py --fuse "" --three 512,256 --nl 0 2>&1 | grep '"fuse": 1' | cut -c1-120
  SRJ_LIB_PATH=build/ab/$v/libsrj.so timeout 300 python tools/coef_class_probe.py 2>&1 | tail -4 | cut -c1-200
done
