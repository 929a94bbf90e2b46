cd $GRAFT_REPO_ROOT
CASCADE_LIB=build/lib_dectrace.so CASCADE_DEC_TRACE=20 timeout 120 python scripts/dbench.py 64 32 2>&1 | grep "decode trace"
timeout 120 python scripts/dbench.py 64 64 2>&1 | tail -1
timeout 120 python scripts/dbench.py 64 64 2>&1 | tail -1
timeout 120 python scripts/dbench.py 64 64 exact 2>&1 | tail -1
timeout 120 python scripts/kbench.py 200 4 2>&1 | tail -6
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python scripts/debug/sanitize_run.py gqa 6 > gpurun_out/sanitize_synccheck_gqa.log 2>&1; echo synccheck gqa rc=$?; grep -E "ERROR SUMMARY|Device Frame" gpurun_out/sanitize_synccheck_gqa.log | sed 's/+0x[0-9a-f]*//' | sort | uniq -c | head -4
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 --timeout-method thread > gpurun_out/pt_g.log 2>&1; echo pytest rc=$?; grep -E "passed|failed|Error" gpurun_out/pt_g.log | tail -3
timeout 600 python scripts/onepass_compare.py 2>&1 | tail -3
