#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 2 --warmup 3 --secondary none --no-cpu --no-e2e > $O/b_torchrun.json 2> $O/b_torchrun.err; echo "torchrun_rc=$?"; head -c 400 $O/b_torchrun.json; echo
python bench.py --steps 2 --warmup 3 --no-e2e --secondary none --no-cpu > $O/b_small.json 2> $O/b_small.err && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --secondary none --no-cpu > $O/ncu_launch.log 2>&1; echo "ncu_launch_rc=$?"
python tools/prof_step.py full --n 32768 --steps 1 > $O/pf_full32k.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dmma_tma_kernel -s 1 -c 1 -o $O/prof_tma_n32768 python tools/prof_step.py full --n 32768 --steps 1 > $O/ncu_tma32k.log 2>&1; echo "ncu_gemm_rc=$?"
python tools/prof_step.py gemv --n 65536 --steps 2 > $O/pf_gemv.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none -k regex:gemv_map_kernel -s 1 -c 1 -o $O/prof_gemv65k python tools/prof_step.py gemv --n 65536 --steps 2 > $O/ncu_gemv.log 2>&1; echo "ncu_gemv_rc=$?"
python tools/prof_step.py spmv --n 2097152 --steps 2 > $O/pf_spmv.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_map_kernel -s 1 -c 1 -o $O/prof_spmv3 python tools/prof_step.py spmv --n 2097152 --steps 2 > $O/ncu_spmv3.log 2>&1; echo "ncu_spmv_rc=$?"
