set -x
python -m pytest tests -m gpu -q -rA -s > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?
python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
for w in 2 4 8; do python bench.py --shard-of $w --steps 3 --warmup 3 --no-decode --no-e2e --no-cpu > gpurun_out/shard$w.json 2> gpurun_out/shard$w.err; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/torchrun1.json 2> gpurun_out/torchrun1.err; echo tr_rc=$?
tail -3 gpurun_out/pytest.log
