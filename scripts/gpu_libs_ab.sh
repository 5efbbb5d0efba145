# A/B of library variants: a short exact-parity subset per library (LIBS),
# then bench.py in MODE (default exact) for each.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for L in ${LIBS:-libfkc_sw}; do
  echo "$L $(FKC_LIB=$PWD/paper_1107_2157_b200/lib/$L.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "${PYTEST_K:-golden or full_size or config2}" 2>&1 | tail -1)"
done
SKIP_TESTS=1 LIBS="${LIBS:-libfkc_sw}" MODE=${MODE:-exact} STEPS=${STEPS:-50} bash scripts/gpu_quick.sh
