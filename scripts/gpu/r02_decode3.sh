timeout 90 python scripts/dbench.py 64 32 2>&1 | tail -1
timeout 90 python scripts/dbench.py 64 32 exact 2>&1 | tail -1
timeout 600 python -m pytest tests -m gpu -q -rA -x -k "decode or gqa or ablation or sharded or errors or degenerate or api or homogeneous or onepass" > gpurun_out/pytest_dec.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|one-pass" gpurun_out/pytest_dec.log | tail -5
