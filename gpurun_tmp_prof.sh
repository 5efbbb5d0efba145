cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for a in "128 2000 fast 0 resident" "128 2000 exact 0 resident" "256 2000 fast 0 resident" "128 2000 fast 0 generic" "256 2000 fast 0 generic"; do timeout 120 python scripts/loop_once.py $a; done > gpurun_out/res_once.txt 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sw_resident -c 1 -o gpurun_out/prof_res128 -f python scripts/loop_once.py 128 200 fast 0 resident > /dev/null 2>&1
cat gpurun_out/res_once.txt
