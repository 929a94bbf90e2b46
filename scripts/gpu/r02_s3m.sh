cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for L in build/lib_coop.so paper_2406_17808_b200/libcascade.so build/lib_coop.so paper_2406_17808_b200/libcascade.so; do
  echo "== $L"; CASCADE_LIB=$L timeout 300 python scripts/kbench.py 200 8 2>&1 | grep -E "maintenance|total"
done
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 --timeout-method thread > gpurun_out/pt_s3m.log 2>&1; echo pytest rc=$?; grep -E "passed|failed|Error" gpurun_out/pt_s3m.log | tail -5
