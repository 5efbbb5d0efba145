# Full GPU round: all gpu tests, smoke, default bench, reference arm,
# ncu launch list + one full capture of each mode of the step kernel, and
# the round's sweeps (resident loop, streamed host run).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu_full.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_full.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_default.txt 2>&1; echo "rc=$?" >> gpurun_out/bench_default.txt
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_reference.txt 2>&1
if [ -z "$SKIP_NCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-other --no-extras > gpurun_out/ncu_launch_bench.txt 2>&1
for m in fast exact; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sw_step_tma -s 12 -c 1 \
     -o gpurun_out/prof_$m -f python bench.py --steps 3 --warmup 10 --no-cpu --no-e2e --no-other --no-extras --mode $m > gpurun_out/ncu_$m.txt 2>&1
done
fi
if [ -z "$SKIP_SWEEPS" ]; then
timeout 900 python scripts/resident_sweep.py --out gpurun_out/resident_sweep.json > gpurun_out/resident_sweep.txt 2>&1
timeout 600 python scripts/stream_timing.py > gpurun_out/stream_timing.txt 2>&1
fi
tail -3 gpurun_out/pytest_gpu_full.txt; tail -1 gpurun_out/smoke.txt; tail -c 1500 gpurun_out/bench_default.txt; tail -c 300 gpurun_out/bench_reference.txt
