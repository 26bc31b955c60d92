cd $GRAFT_REPO_ROOT
for nf in "" 1; do
  echo "NOFLAGS=$nf"
  for c in "cfg5 32 256 256 --fuse 2 --steps 1600" "cfg2 512 4096 --fuse 4 --steps 4000" "cfg3 64 512 512 --fuse 2 --steps 800"; do
    if [ -n "$nf" ]; then export SRJ_SLAB_NOFLAGS=1; else unset SRJ_SLAB_NOFLAGS; fi
    timeout 300 python - <<PY
import sys, json
sys.path.insert(0, "tools")
import slab_rank_probe as s
a = "$c".split()
own = [int(x) for x in a[1:a.index("--fuse")]]
r = s.probe(a[0], own, int(a[a.index("--fuse")+1]), int(a[a.index("--steps")+1]), 3, modes=("direct_store",))
print(json.dumps(r))
PY
  done
done
