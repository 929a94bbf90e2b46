set -x
python -m pytest tests -m gpu -q -rA -x -k "decode or gqa or ablation or sharded or errors or smoke or degenerate" > gpurun_out/pytest_dec.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_dec.log
python scripts/dbench.py > gpurun_out/dbench.txt 2>&1; echo dbench_rc=$?
tail -5 gpurun_out/dbench.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-decode > gpurun_out/torchrun1.json 2> gpurun_out/torchrun1.err; echo tr_rc=$?
head -c 300 gpurun_out/torchrun1.json
