cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_dist_nccl.py tests/test_gpu_api.py -m gpu -q -x --timeout 300 --timeout-method thread 2>&1 | tail -5
