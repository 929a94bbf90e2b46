# round-2 re-entry: full GPU suite + default bench + decode bench
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -rA -x > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/pytest.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
tail -3 gpurun_out/bench.err; cut -c1-600 gpurun_out/bench.json
timeout 300 python bench.py --steps 3 --warmup 3 --score-mode onepass --no-decode --no-e2e --no-cpu > gpurun_out/bench_onepass.json 2> gpurun_out/bench_onepass.err; echo bench1p_rc=$?
cut -c1-400 gpurun_out/bench_onepass.json
