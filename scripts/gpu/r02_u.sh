cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_api.py tests/test_gpu_stack.py tests/test_gpu_dist_nccl.py -m gpu -q -x --timeout 600 --timeout-method thread 2>&1 | tail -3
