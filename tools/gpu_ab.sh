cd $GRAFT_REPO_ROOT
# A/B timing of libsrj builds under build/ab/*/ (args: variant names)
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv -lms 500 > gpurun_out/ab_clocks.csv &
SMI=$!
for rep in 1 2; do for v in "$@"; do
  SRJ_LIB_PATH=build/ab/$v/libsrj.so timeout 300 python tools/probe3d.py ${PROBE_ARGS} | sed "s/^/$v /" >> gpurun_out/ab.log
done; done
kill $SMI
cat gpurun_out/ab.log | python -c "
import sys,json
for l in sys.stdin:
  v,j=l.split(' ',1); d=json.loads(j); print(v, d['workload'], d['n'], round(d['glups'],1), d['sha1'][:10])"
