# One ncu --set full capture of the step kernel (fast mode unless MODE set;
# TAG names the output, BENCH_ARGS go to bench.py) plus the per-SASS-
# instruction source page, for offline analysis here.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
M=${MODE:-fast}
T=${TAG:-$M}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sw_step_tma -s 12 -c 1 \
   -o gpurun_out/prof_$T -f python bench.py --steps 3 --warmup 10 --no-cpu --no-e2e --no-other --no-extras --mode $M ${BENCH_ARGS} > gpurun_out/ncu_$T.txt 2>&1
ncu -i gpurun_out/prof_$T.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$T.csv 2>&1
tail -2 gpurun_out/ncu_$T.txt; wc -l gpurun_out/src_$T.csv
