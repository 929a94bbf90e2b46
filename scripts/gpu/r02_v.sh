cd $GRAFT_REPO_ROOT
for lib in paper_2406_17808_b200/libcascade.so build/lib_fe3.so build/lib_fe5.so paper_2406_17808_b200/libcascade.so build/lib_fe3.so build/lib_fe5.so; do
  echo "== $lib"; CASCADE_LIB=$lib timeout 120 python scripts/kbench.py 200 8 2>&1 | grep -E "attn_fwd"
done
