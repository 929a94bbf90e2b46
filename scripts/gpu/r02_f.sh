cd $GRAFT_REPO_ROOT
CASCADE_LIB=build/lib_dectrace.so CASCADE_DEC_TRACE=20 timeout 120 python scripts/dbench.py 64 32 2>&1 | tail -22
timeout 120 python scripts/dbench.py 64 64 2>&1 | tail -1
timeout 120 python scripts/kbench.py 200 4 2>&1 | tail -6
for w in gqa toy; do
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python scripts/debug/sanitize_run.py $w 6 > gpurun_out/sanitize_synccheck_$w.log 2>&1; echo synccheck $w rc=$?; grep -E "ERROR SUMMARY|Device Frame" gpurun_out/sanitize_synccheck_$w.log | sed 's/+0x[0-9a-f]*//' | sort | uniq -c | head -4
done
timeout 1200 python -m pytest tests -m gpu -q -x -k "parity or closure or onepass or stack" --timeout 900 --timeout-method thread > gpurun_out/pt_f.log 2>&1; echo pytest rc=$?; grep -E "passed|failed|Error" gpurun_out/pt_f.log | tail -3
