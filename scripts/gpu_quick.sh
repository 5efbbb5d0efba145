# Quick GPU loop: parity tests (optionally -k filtered; SKIP_TESTS=1 skips),
# then a bench sweep over LIBS x DIAGS x ALTS x SEGS (fast mode unless MODE),
# optionally with the ncu DRAM traffic / duration of each config (NCU=1).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
if [ -z "$SKIP_TESTS" ]; then
timeout 1200 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_quick.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.txt
tail -4 gpurun_out/pytest_quick.txt
fi
: > gpurun_out/quick_sweep.txt
for lib in ${LIBS:-libfkc_sw}; do for diag in ${DIAGS:-none}; do for alt in ${ALTS:-1}; do for seg in ${SEGS:-0}; do
  export FKC_LIB=$PWD/paper_1107_2157_b200/lib/$lib.so
  echo "$lib diag=$diag alt=$alt seg=$seg $(timeout 300 python bench.py --steps ${STEPS:-200} --warmup 10 --no-cpu --no-e2e --no-other --mode ${MODE:-fast} --seg $seg --alt $alt --diag $diag 2>&1 | tail -1 | python3 -c 'import json,sys
try:
  d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
except Exception as e: print("ERR", e)')" >> gpurun_out/quick_sweep.txt
  if [ -n "$NCU" ]; then
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:sw_step_tma -s 5 -c 1 --csv \
    python bench.py --steps 2 --warmup 5 --no-cpu --no-e2e --no-other --mode ${MODE:-fast} --seg $seg --alt $alt --diag $diag > gpurun_out/ncu_q.csv 2>&1
  echo "   ncu: $(grep -E 'dram__bytes|gpu__time' gpurun_out/ncu_q.csv | awk -F'","' '{print $(NF-2)"="$NF}' | tr -d '"' | tr '\n' ' ')" >> gpurun_out/quick_sweep.txt
  fi
done; done; done; done
cat gpurun_out/quick_sweep.txt
