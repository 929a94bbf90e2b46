cd $GRAFT_REPO_ROOT
CASCADE_LIB=build/lib_dectrace.so CASCADE_DEC_TRACE=20 timeout 120 python scripts/dbench.py 64 32 2>&1 | grep "decode trace"
timeout 120 python scripts/dbench.py 64 64 2>&1 | tail -1
timeout 120 python scripts/dbench.py 64 64 2>&1 | tail -1
timeout 120 python scripts/dbench.py 64 64 exact 2>&1 | tail -1
timeout 1200 python -m pytest tests -m gpu -q -x -k "decode or gqa or api or ablation or sharded or homogeneous or cfg4" --timeout 900 --timeout-method thread > gpurun_out/pt_n.log 2>&1; echo pytest rc=$?; grep -E "passed|failed|Error" gpurun_out/pt_n.log | tail -3
