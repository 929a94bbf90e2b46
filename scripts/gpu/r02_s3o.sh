cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
CASCADE_MAINT_TRACE=204 timeout 300 python scripts/kbench.py 200 4 > gpurun_out/mtrace_comp.txt 2>&1
CASCADE_LIB=build/lib_coop.so CASCADE_MAINT_TRACE=204 timeout 300 python scripts/kbench.py 200 4 > gpurun_out/mtrace_coop.txt 2>&1
head -3 gpurun_out/mtrace_comp.txt; grep -c . gpurun_out/mtrace_comp.txt
