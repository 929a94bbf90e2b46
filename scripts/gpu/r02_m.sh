cd $GRAFT_REPO_ROOT
export CASCADE_PASS1_SPLIT=1
timeout 120 python scripts/debug/sanitize_run.py gqa 6 2>&1 | tail -2
timeout 120 python scripts/kbench.py 200 6 2>&1 | grep -E "attn_fwd|total"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_closure.py -m gpu -q -x --timeout 600 --timeout-method thread > gpurun_out/pt_m.log 2>&1; echo pytest rc=$?; grep -E "passed|failed|Error|assert" gpurun_out/pt_m.log | head -8
unset CASCADE_PASS1_SPLIT
timeout 120 python scripts/kbench.py 200 6 2>&1 | grep -E "attn_fwd|total"
