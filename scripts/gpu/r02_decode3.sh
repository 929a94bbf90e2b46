timeout 300 python scripts/dbench.py 64 32 2>&1 | tail -1
timeout 300 python scripts/dbench.py 64 32 exact 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -rA -x -k "decode or gqa or ablation or sharded or errors or degenerate or api or homogeneous" > gpurun_out/pytest_dec.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_dec.log
