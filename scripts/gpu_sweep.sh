# Variant sweep: alternative builds of the library (FKC_LIB) x mode.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "not 16384 and not config2" > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
: > gpurun_out/sweep.txt
one() { # label, env, args
  echo "$1 $(env $2 timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e $3 2>&1 | tail -1 | python3 -c 'import json,sys
try:
  d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"])
except Exception as e: print("ERR", e)')" >> gpurun_out/sweep.txt
}
for lib in libfkc_sw libfkc_sw_unr2 libfkc_sw_fixup; do
  one "exact $lib" "FKC_LIB=$PWD/paper_1107_2157_b200/lib/$lib.so" "--mode exact"
done
one "fast default" "X=1" "--mode fast"
tail -2 gpurun_out/pytest_gpu.txt; cat gpurun_out/sweep.txt
