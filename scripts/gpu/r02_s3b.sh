cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for L in paper_2406_17808_b200/libcascade.so build/lib_pipe.so build/lib_pipe_e3.so build/lib_pipe_e5.so build/lib_pipe_e6.so build/lib_pipe.so paper_2406_17808_b200/libcascade.so; do
  echo "== $L"; CASCADE_LIB=$L timeout 300 python scripts/kbench.py 200 6 2>&1 | grep -E "attn_score|attn_fwd|total"
done
CASCADE_LIB=build/lib_pipe.so timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 --timeout-method thread > gpurun_out/pt_s3b_pipe.log 2>&1; echo pipe pytest rc=$?; grep -E "passed|failed|Error" gpurun_out/pt_s3b_pipe.log | tail -3
