#!/bin/bash
# GPU box script: tests, timings, then ncu captures (each after a clean plain run).
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -q 2>&1 > $O/pytest_gpu2.log; echo "pytest_rc=$?"; tail -5 $O/pytest_gpu2.log
for w in "full --n 8192" "full --n 32768 --steps 1" "gemv --n 65536" "spmv --n 2097152"; do timeout 300 python tools/prof_step.py $w --steps 5 2>&1 | tail -1; done
python tools/prof_step.py full --n 8192 --steps 2 > $O/pf_full.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:dmma_gemm_kernel -s 1 -c 1 -o $O/prof_gemm_n8192 python tools/prof_step.py full --n 8192 --steps 2 > $O/ncu_gemm.log 2>&1; echo "ncu_gemm_rc=$?"
python tools/prof_step.py spmv --n 2097152 --steps 2 > $O/pf_spmv.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_map_kernel -s 1 -c 1 -o $O/prof_spmv python tools/prof_step.py spmv --n 2097152 --steps 2 > $O/ncu_spmv.log 2>&1; echo "ncu_spmv_rc=$?"
python tools/prof_step.py gemv --n 32768 --steps 2 > $O/pf_gemv.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv_map_kernel -s 1 -c 1 -o $O/prof_gemv python tools/prof_step.py gemv --n 32768 --steps 2 > $O/ncu_gemv.log 2>&1; echo "ncu_gemv_rc=$?"
python bench.py --steps 2 --warmup 3 --no-e2e --secondary none --no-cpu > $O/b_small.json 2> $O/b_small.err && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --secondary none --no-cpu > $O/ncu_launch.log 2>&1; echo "ncu_launch_rc=$?"
ls -la $O
