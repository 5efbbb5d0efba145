# GPU round trip: tests, benches, ncu launch list + full capture.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "not 16384 and not config2" > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
for m in exact fast; do
  timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e --mode $m > gpurun_out/bench_$m.txt 2>&1
done
for m in exact fast; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sw_step_tma -s 4 -c 1 \
     -o gpurun_out/prof_$m -f python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --mode $m > gpurun_out/ncu_$m.txt 2>&1
done
tail -3 gpurun_out/pytest_gpu.txt; for f in gpurun_out/bench_*.txt; do tail -c 600 $f; echo; done
