cd $GRAFT_REPO_ROOT
for lib in "" build/lib_r2p2.so build/lib_r3p1.so build/lib_r2p1.so; do
  echo "== decode lib=${lib:-default}"
  CASCADE_LIB=$lib timeout 120 python scripts/dbench.py 64 64 2>&1 | tail -1
  CASCADE_LIB=$lib timeout 120 python scripts/dbench.py 64 64 2>&1 | tail -1
done
timeout 120 python scripts/dbench.py 64 64 exact 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x -k "decode or gqa or sharded or homogeneous or api or ablation or stack" --timeout 600 --timeout-method thread > gpurun_out/pt_c.log 2>&1; echo pytest rc=$?; grep -E "passed|failed|Error" gpurun_out/pt_c.log | tail -3
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python scripts/debug/sanitize_run.py gqa 6 > gpurun_out/sanitize_synccheck_gqa.log 2>&1; echo synccheck gqa rc=$?; tail -2 gpurun_out/sanitize_synccheck_gqa.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/debug/sanitize_run.py gqa 6 > gpurun_out/sanitize_memcheck_gqa.log 2>&1; echo memcheck gqa rc=$?; tail -2 gpurun_out/sanitize_memcheck_gqa.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python scripts/debug/sanitize_run.py gqa 3 > gpurun_out/sanitize_racecheck_gqa.log 2>&1; echo racecheck gqa rc=$?; tail -2 gpurun_out/sanitize_racecheck_gqa.log
