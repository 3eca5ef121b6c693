#!/bin/bash
# Round-end regression on one B200: smoke, pytest -m gpu, bench (default), the ncu launch
# list of a short bench run (each after its own command exited 0 without ncu).
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke_rc=$?"; tail -1 $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest_rc=$?"; tail -2 $O/pytest_gpu.log; grep -E "^FAILED" $O/pytest_gpu.log | head -20
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; rc=$?; echo "bench_rc=$rc"; tail -c 300 $O/bench.err
if [ "$rc" = 0 ] && [ "${NCU:-1}" = 1 ]; then
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --secondary none --no-cpu > $O/ncu_bench.log 2>&1; echo "ncu_rc=$?"
fi
