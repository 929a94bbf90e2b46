cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for i in 1 2 3; do CASCADE_LIB=build/lib_obs1.so timeout 300 python scripts/kbench.py 200 8 2>&1 | grep -E "attn_fwd" | sed 's/^/old /'; timeout 300 python scripts/kbench.py 200 8 2>&1 | grep -E "attn_fwd|total" | sed 's/^/new /'; done
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python scripts/debug/sanitize_run.py gqa 6 > gpurun_out/san_sync_s3v.log 2>&1; echo synccheck gqa rc=$?; grep -E "ERROR SUMMARY" gpurun_out/san_sync_s3v.log | tail -2
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python scripts/debug/sanitize_run.py cfg2 3 > gpurun_out/san_sync2_s3v.log 2>&1; echo synccheck cfg2 rc=$?; grep -E "ERROR SUMMARY" gpurun_out/san_sync2_s3v.log | tail -2
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 --timeout-method thread > gpurun_out/pt_s3v.log 2>&1; echo pytest rc=$?; grep -E "passed|failed|Error" gpurun_out/pt_s3v.log | tail -3
