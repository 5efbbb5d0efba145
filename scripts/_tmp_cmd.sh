cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
P='import sys,json
for l in sys.stdin:
  try: d=json.loads(l); print(d["mode"], d["n"], "seg", d["seg"], "w", d["warps"], d["gcell_s"])
  except Exception: print(l.rstrip()[:200])'
for m in fast exact; do
timeout 900 python scripts/grid_sweep.py --mode $m --sizes 1024,1448,2048,2896 --variants tma --warps 0 --segs 0,6,10,14,22 2>&1 | python3 -c "$P"
done
