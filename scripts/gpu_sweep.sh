# Sweep: library build variants (FKC_LIB) x TMA row-segment length, fast mode.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/sweep.txt
one() { # label, env, args
  echo "$1 $(env $2 timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu --no-e2e --no-other $3 2>&1 | tail -1 | python3 -c 'import json,sys
try:
  d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
except Exception as e: print("ERR", e)')" >> gpurun_out/sweep.txt
}
for lib in ${LIBS:-libfkc_sw}; do
for seg in ${SEGS:-96 128 256}; do one "$lib seg=$seg ${MODE:-fast}" "FKC_LIB=$PWD/paper_1107_2157_b200/lib/$lib.so" "--mode ${MODE:-fast} --seg $seg"; done
done
cat gpurun_out/sweep.txt
