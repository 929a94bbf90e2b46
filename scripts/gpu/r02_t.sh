cd $GRAFT_REPO_ROOT
timeout 120 python scripts/debug/onepass_dbg.py 128 8 2>&1 | tail -3
timeout 120 python scripts/kbench.py 200 6 4096 onepass 2>&1 | grep -E "attn_fwd|total"
timeout 120 python scripts/kbench.py 200 6 2>&1 | grep -E "attn_fwd|total"
timeout 1200 python -m pytest tests/test_gpu_closure.py tests/test_gpu_parity.py -m gpu -q -x --timeout 600 --timeout-method thread > gpurun_out/pt_t.log 2>&1; echo pytest rc=$?; grep -E "passed|failed|Error|one-pass" gpurun_out/pt_t.log | tail -4
timeout 300 python bench.py --steps 3 --warmup 3 --score-mode onepass --no-decode --no-e2e --no-cpu > gpurun_out/bench_onepass2.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/bench_onepass2.json')); print('onepass bench', round(d['value']), d['kernels'])"
