cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out; mkdir -p $O
df -h /dev/shm | tail -1
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest_rc=$?"; tail -8 $O/pytest_gpu.log
IPT_PROFILE=1 timeout 300 python tools/profile_config5_e2e.py 2>&1 | tail -5
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench_rc=$?"; tail -c 600 $O/bench.err
