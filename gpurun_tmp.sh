cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
L=$PWD/paper_1107_2157_b200/lib
for lib in libfkc_sw libfkc_sw_xu2 libfkc_sw_xu2w8 libfkc_sw_xw8; do
  for diag in none cfl; do
  export FKC_LIB=$L/$lib.so
  echo "$lib diag=$diag $(timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e --no-other --no-extras --mode exact --diag $diag 2>&1 | grep '^{' | python3 -c 'import json,sys
d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"])')"
  done
done > gpurun_out/exact_var.txt 2>&1
cat gpurun_out/exact_var.txt
