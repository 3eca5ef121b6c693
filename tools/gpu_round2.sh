#!/bin/bash
# Round-2 regression on one B200: smoke, pytest -m gpu, bench, then one compute-sanitizer
# tool at a time on the smoke-size workload (tools/sanitize_smoke.py).
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke_rc=$?"; tail -2 $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest_rc=$?"; tail -3 $O/pytest_gpu.log; grep -E "^FAILED" $O/pytest_gpu.log | head -20
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench_rc=$?"; tail -c 300 $O/bench.err
if [ "${SANITIZE:-1}" = 1 ]; then
  for t in memcheck racecheck synccheck initcheck; do
    timeout 1200 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_smoke.py > $O/sanitize_$t.log 2>&1
    echo "sanitize_${t}_rc=$?"; tail -3 $O/sanitize_$t.log
  done
fi
