# resident-loop timing (scripts/debug_resident.py) for each library in LIBS
cd $GRAFT_REPO_ROOT
for L in ${LIBS:-libfkc_sw}; do
  echo "== $L"
  FKC_LIB=$PWD/paper_1107_2157_b200/lib/$L.so python scripts/debug_resident.py 2>&1 | grep -E "differing \[[1-9]|steps=1000"
done
