cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for L in paper_2406_17808_b200/libcascade.so build/lib_desync.so paper_2406_17808_b200/libcascade.so build/lib_desync.so; do
  echo "== $L"; CASCADE_LIB=$L timeout 300 python scripts/dbench.py 64 128 2>&1 | tail -1
done
CASCADE_LIB=build/lib_desync.so timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 --timeout-method thread -k "decode" > gpurun_out/pt_s3t.log 2>&1; echo desync decode pytest rc=$?; grep -E "passed|failed|Error" gpurun_out/pt_s3t.log | tail -3
