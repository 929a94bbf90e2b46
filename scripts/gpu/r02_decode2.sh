set -x
python -m pytest tests -m gpu -q -rA -x -k "decode or gqa or ablation or sharded or errors or degenerate or api or homogeneous" > gpurun_out/pytest_dec.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_dec.log
python scripts/dbench.py > gpurun_out/dbench.txt 2>&1; echo dbench_rc=$?
tail -2 gpurun_out/dbench.txt
timeout 900 ncu --set full --import-source on -k regex:decode_fused -s 3 -c 1 -o gpurun_out/dec_fused_v3 -f python scripts/dbench.py 64 6 > gpurun_out/ncu_dec.log 2>&1; echo ncu_rc=$?
tail -3 gpurun_out/ncu_dec.log
