cd $GRAFT_REPO_ROOT
timeout 120 python scripts/kbench.py 200 4 2>&1 | grep -E "prep|total"
CASCADE_LIB=build/lib_prep4.so timeout 120 python scripts/kbench.py 200 4 2>&1 | grep -E "prep|total"
git_prev=1
timeout 1800 python -m pytest tests -m gpu -q -x -k "parity or closure or fullsize" --timeout 900 --timeout-method thread > gpurun_out/pt_j.log 2>&1; echo pytest rc=$?; grep -E "passed|failed|Error" gpurun_out/pt_j.log | tail -3
