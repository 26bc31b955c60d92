cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/ab2d.log
bash tools/gpu_ab2d.sh before after > /dev/null 2>&1
cat gpurun_out/ab2d.log
for rep in 1 2; do for v in before after; do
  echo $v; SRJ_LIB_PATH=build/ab/$v/libsrj.so timeout 300 python tools/probe3d.py 2>&1 | cut -c1-110
done; done
