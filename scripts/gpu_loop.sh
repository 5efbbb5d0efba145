# Persistent-loop round: its GPU tests, then the loop sweep (LOOP_ARGS).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_loop.py -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_loop.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_loop.txt
tail -15 gpurun_out/pytest_loop.txt
timeout 1200 python scripts/loop_sweep.py $LOOP_ARGS --out gpurun_out/loop_sweep.json > gpurun_out/loop_sweep.txt 2>&1
echo "sweep rc=$?" >> gpurun_out/loop_sweep.txt
cat gpurun_out/loop_sweep.txt | tail -40
