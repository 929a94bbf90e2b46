cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
CASCADE_LIB=build/lib_p2t.so timeout 300 python scripts/kbench.py 200 32 2>&1 | grep -E "pass2 trace|attn_score" | tail -4
