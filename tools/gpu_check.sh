#!/bin/bash
# Full GPU regression: smoke, pytest -m gpu, reference harness, API latency.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1800 python -m pytest tests -m gpu -q 2>&1 > $O/pytest_gpu.log; echo "pytest_rc=$?"; tail -4 $O/pytest_gpu.log
[ -x tools/cpp/api_latency ] && ./tools/cpp/api_latency 1024 2>&1 | tail -2
[ -x tools/cpp/api_latency ] && ./tools/cpp/api_latency 256 2>&1 | tail -1
grep -E "PASS|FAIL" $O/pytest_gpu.log | head -20
