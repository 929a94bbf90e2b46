cd $GRAFT_REPO_ROOT
export CUDA_LAUNCH_BLOCKING=1
timeout 60 python scripts/debug/onepass_dbg.py 128 8 2>&1 | tail -12; echo rc=$?
timeout 60 python scripts/debug/onepass_dbg.py 64 4 2>&1 | tail -12; echo rc=$?
unset CUDA_LAUNCH_BLOCKING
timeout 120 compute-sanitizer --tool memcheck python scripts/debug/onepass_dbg.py 128 8 2>&1 | tail -30
timeout 120 python scripts/dbench.py 64 32 2>&1 | tail -2
for f in test_gpu_api test_gpu_kernels test_gpu_parity; do
  timeout 900 python -m pytest tests/$f.py -m gpu -q -x -p pytest_timeout --timeout 300 --timeout-method thread > gpurun_out/pt_$f.log 2>&1; echo $f rc=$?; tail -3 gpurun_out/pt_$f.log
done
timeout 900 python -m pytest tests/test_gpu_closure.py -m gpu -q -x -k "not onepass" -p pytest_timeout --timeout 300 --timeout-method thread > gpurun_out/pt_closure.log 2>&1; echo closure rc=$?; tail -3 gpurun_out/pt_closure.log
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -p pytest_timeout --timeout 600 --timeout-method thread > gpurun_out/pt_full.log 2>&1; echo full rc=$?; tail -3 gpurun_out/pt_full.log
