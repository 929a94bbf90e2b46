cd $GRAFT_REPO_ROOT
timeout 120 python scripts/dbench.py 64 64 2>&1 | tail -1
timeout 120 python scripts/dbench.py 64 64 2>&1 | tail -1
timeout 120 python scripts/dbench.py 64 64 exact 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x -k "decode or gqa or sharded or homogeneous or api or ablation" --timeout 600 --timeout-method thread > gpurun_out/pt_d.log 2>&1; echo pytest rc=$?; grep -E "passed|failed|Error" gpurun_out/pt_d.log | tail -3
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python scripts/debug/sanitize_run.py gqa 6 > gpurun_out/sanitize_synccheck_gqa.log 2>&1; echo synccheck gqa rc=$?; grep -E "ERROR SUMMARY|Device Frame" gpurun_out/sanitize_synccheck_gqa.log | sed 's/+0x[0-9a-f]*//' | sort | uniq -c | head
