# ncu: the 2048^2 fast CFL step with dt fixed vs dt from the bound row
# (scripts/red_cost.py --eager): per-kernel duration and a full capture each.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=${N:-2048}
for c in all_cfl all_cfl_bound; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sw_step_tma -s 6 -c 1 \
     -o gpurun_out/prof_$c -f python scripts/red_cost.py --sizes $N --modes fast --combos $c --eager 10 > gpurun_out/ncu_$c.txt 2>&1
  tail -1 gpurun_out/ncu_$c.txt
done
