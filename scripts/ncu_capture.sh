# One ncu --set full capture of the step kernel (fast mode unless MODE set)
# plus the per-SASS-instruction source page, for offline analysis here.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
M=${MODE:-fast}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sw_step_tma -s 12 -c 1 \
   -o gpurun_out/prof_$M -f python bench.py --steps 3 --warmup 10 --no-cpu --no-e2e --no-other --mode $M ${BENCH_ARGS} > gpurun_out/ncu_$M.txt 2>&1
ncu -i gpurun_out/prof_$M.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$M.csv 2>&1
tail -2 gpurun_out/ncu_$M.txt; wc -l gpurun_out/src_$M.csv
