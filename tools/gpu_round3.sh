#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out
for w in "full --n 8192" "full --n 32768 --steps 2" "gemv --n 65536" "spmv --n 2097152"; do timeout 300 python tools/prof_step.py $w --steps 5 2>&1 | tail -1; done
timeout 900 ./oracle/_ref/unit_b200 > $O/unit_b200.log 2>&1; echo "unit_rc=$?"; tail -3 $O/unit_b200.log; grep FAIL $O/unit_b200.log | head
timeout 1800 ./oracle/_ref/acceptance_b200 > $O/acceptance_b200.log 2>&1; echo "acc_rc=$?"; cat $O/acceptance_b200.log
timeout 900 python -m pytest tests/test_gpu_full.py -q -x 2>&1 | tail -3
python tools/prof_step.py full --n 32768 --steps 1 > $O/pf_full32k.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dmma_gemm_kernel -s 1 -c 1 -o $O/prof_gemm_n32768 python tools/prof_step.py full --n 32768 --steps 1 > $O/ncu_gemm32k.log 2>&1; echo "ncu_gemm_rc=$?"
python tools/prof_step.py spmv --n 2097152 --steps 2 > $O/pf_spmv.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_map_kernel -s 1 -c 1 -o $O/prof_spmv2 python tools/prof_step.py spmv --n 2097152 --steps 2 > $O/ncu_spmv2.log 2>&1; echo "ncu_spmv_rc=$?"
