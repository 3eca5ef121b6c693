cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_local_ranks.py tests/test_gpu_single.py tests/test_gpu_row_blocks.py -q -x > $O/single.log 2>&1; echo "single_rc=$?"; tail -15 $O/single.log
timeout 300 python tools/row_shard_probe.py 2>&1 | tail -4
timeout 300 python tools/spmv_probe.py > $O/spmv_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmv_group -s 45 -c 1 -o $O/prof_spmv_r02c python tools/spmv_probe.py > $O/ncu_spmv.log 2>&1; echo "ncu_rc=$?"; tail -1 $O/spmv_plain.log
