cd $GRAFT_REPO_ROOT
timeout 60 python scripts/debug/onepass_dbg.py 128 8 2>&1 | tail -9; echo rc=$?
timeout 60 python scripts/debug/onepass_dbg.py 64 4 2>&1 | tail -3; echo rc=$?
timeout 300 python -m pytest tests/test_gpu_stack.py -m gpu -q -x -s --timeout 240 --timeout-method thread > gpurun_out/pt_stack.log 2>&1; echo stack rc=$?; tail -5 gpurun_out/pt_stack.log
for f in test_gpu_api test_gpu_kernels test_gpu_parity test_gpu_closure; do
  timeout 1200 python -m pytest tests/$f.py -m gpu -q -x -s --timeout 400 --timeout-method thread > gpurun_out/pt_$f.log 2>&1; echo $f rc=$?; grep -E "passed|failed|one-pass" gpurun_out/pt_$f.log | tail -3
done
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -s --timeout 900 --timeout-method thread > gpurun_out/pt_full.log 2>&1; echo full rc=$?; tail -3 gpurun_out/pt_full.log
timeout 300 python bench.py --steps 3 --warmup 3 --score-mode onepass --no-decode --no-e2e --no-cpu > gpurun_out/bench_onepass.json 2> gpurun_out/bench_onepass.err; echo bench1p_rc=$?
cut -c1-300 gpurun_out/bench_onepass.json
