cd $GRAFT_REPO_ROOT
timeout 120 python scripts/kbench.py 200 6 2>&1 | grep -E "ms/chunk|total"
timeout 120 python scripts/dbench.py 64 64 2>&1 | tail -1
CASCADE_NVTX=1 timeout 300 ncu --nvtx --nvtx-include "cascade.maintenance/" --metrics gpu__time_duration.sum -c 2 python scripts/debug/sanitize_run.py gqa 4 2>&1 | grep -E "maint_coop|NVTX|gpu__time" | head -6
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 --timeout-method thread > gpurun_out/pt_r.log 2>&1; echo pytest rc=$?; grep -E "passed|failed|Error" gpurun_out/pt_r.log | tail -3
