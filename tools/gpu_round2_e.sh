cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out; mkdir -p $O
free -g | head -2; nproc
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest_rc=$?"; tail -8 $O/pytest_gpu.log
IPT_PROFILE=1 timeout 300 python tools/profile_config5_e2e.py 2>&1 | tail -20
timeout 600 ./tools/cpp/dropin_bench 2 3 2>&1 | tail -2
timeout 600 ./tools/cpp/dropin_bench 5 3 2>&1 | tail -2
timeout 900 ./tools/cpp/dropin_bench 3 2 2>&1 | tail -2
