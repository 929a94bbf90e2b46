cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for L in build/lib_s0e0.so paper_2406_17808_b200/libcascade.so build/lib_s1e0.so build/lib_s0e1.so build/lib_emu6.so build/lib_emu2.so build/lib_s0e0.so paper_2406_17808_b200/libcascade.so; do
  echo "== $L"; CASCADE_LIB=$L timeout 300 python scripts/kbench.py 200 6 2>&1 | grep -E "attn_score|total"
done
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 --timeout-method thread > gpurun_out/pt_s3d.log 2>&1; echo pytest rc=$?; grep -E "passed|failed|Error" gpurun_out/pt_s3d.log | tail -3
