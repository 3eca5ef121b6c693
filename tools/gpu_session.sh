cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest_rc=$?"; tail -6 $O/pytest_gpu.log; grep -E "^FAILED|Error" $O/pytest_gpu.log | head -20
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench_rc=$?"; tail -c 400 $O/bench.err
