cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_local_ranks.py -x -q > $O/local_ranks.log 2>&1; echo "local_rc=$?"; tail -15 $O/local_ranks.log
timeout 300 python tools/spmv_probe.py > $O/spmv_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmv_group -s 10 -c 2 -o $O/prof_spmv_r02 python tools/spmv_probe.py > $O/ncu_spmv.log 2>&1; echo "ncu_rc=$?"; cat $O/spmv_plain.log | tail -2
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest_rc=$?"; tail -5 $O/pytest_gpu.log
