# ncu --set full of the resident time-loop kernel (N^2 grid, MODE), plus the
# per-SASS source page for offline analysis.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=${N:-128}; M=${MODE:-fast}; T=${TAG:-res_${M}_${N}}
cat > /tmp/res_run.py <<PY
import sys; sys.path.insert(0, ".")
import torch
from paper_1107_2157_b200 import swdemo
cfg = swdemo.SWConfig(nx=$N, ny=$N, dt=0.01, variant="resident", mode="$M")
sim = swdemo.Simulation(cfg, state=swdemo.init_state(cfg), diagnostics=False)
sim.advance(200)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sw_resident -c 1 -o gpurun_out/prof_$T -f python /tmp/res_run.py > gpurun_out/ncu_$T.txt 2>&1
ncu -i gpurun_out/prof_$T.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$T.csv 2>&1
tail -2 gpurun_out/ncu_$T.txt
