cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for L in paper_2406_17808_b200/libcascade.so build/lib_obs2.so build/lib_obs0.so paper_2406_17808_b200/libcascade.so build/lib_obs2.so build/lib_obs0.so; do
  echo "== $L"; CASCADE_LIB=$L timeout 300 python scripts/kbench.py 200 8 2>&1 | grep -E "attn_fwd"
done
