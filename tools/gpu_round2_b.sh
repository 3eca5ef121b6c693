cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_local_ranks.py tests/test_gpu_warm_complex.py -q > $O/local_ranks.log 2>&1; echo "local_rc=$?"; tail -25 $O/local_ranks.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest_rc=$?"; tail -8 $O/pytest_gpu.log
