# compute-sanitizer over the library's kernels (scripts/sanitize.py workload).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/sanitize.txt
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  timeout 1200 compute-sanitizer --tool $tool --target-processes all --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize workload done' gpurun_out/sanitize_$tool.txt | tr '\n' ' ')" >> gpurun_out/sanitize.txt
done
cat gpurun_out/sanitize.txt
