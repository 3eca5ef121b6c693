#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_full.py tests/test_gpu_large.py -q -x -k "not config3" 2>&1 | tail -3
for w in "full --n 8192" "full --n 16384 --steps 3" "full --n 32768 --steps 2"; do timeout 300 python tools/prof_step.py $w --steps 5 2>&1 | tail -1; done
python tools/prof_step.py full --n 8192 --steps 2 > $O/pf_full.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:dmma_tma_kernel -s 1 -c 1 -o $O/prof_tma2_n8192 python tools/prof_step.py full --n 8192 --steps 2 > $O/ncu_tma.log 2>&1; echo "ncu_rc=$?"
