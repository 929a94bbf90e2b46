cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for L in build/lib_old.so paper_2406_17808_b200/libcascade.so build/lib_mb6.so build/lib_mb8.so build/lib_old.so paper_2406_17808_b200/libcascade.so; do
  echo "== $L"; CASCADE_LIB=$L timeout 300 python scripts/kbench.py 200 8 2>&1 | grep -E "prep"
done
