#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_full.py -q -x 2>&1 | tail -5
for w in "full --n 8192" "full --n 32768 --steps 2"; do timeout 300 python tools/prof_step.py $w --steps 5 2>&1 | tail -1; done
timeout 900 ./oracle/_ref/acceptance_b200 > $O/acceptance_b200.log 2>&1; echo "acc_rc=$?"; cat $O/acceptance_b200.log
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5
python tools/prof_step.py full --n 8192 --steps 2 > $O/pf_full.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:dmma_tma_kernel -s 1 -c 1 -o $O/prof_tma_n8192 python tools/prof_step.py full --n 8192 --steps 2 > $O/ncu_tma.log 2>&1; echo "ncu_rc=$?"
