cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for L in paper_2406_17808_b200/libcascade.so build/lib_ks.so build/lib_ks_e2.so build/lib_ks_e6.so build/lib_ks.so paper_2406_17808_b200/libcascade.so; do
  echo "== $L"; CASCADE_LIB=$L timeout 300 python scripts/kbench.py 200 6 2>&1 | grep -E "attn_fwd|total"
done
CASCADE_LIB=build/lib_ks.so timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 --timeout-method thread > gpurun_out/pt_s3j_ks.log 2>&1; echo ks pytest rc=$?; grep -E "passed|failed|Error" gpurun_out/pt_s3j_ks.log | tail -5
