cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out; mkdir -p $O
for v in 9 16 17 9 16 17; do IPT_SPMV_VARIANT=$v timeout 300 python tools/spmv_probe.py 2>&1 | tail -1; done
IPT_SPMV_VARIANT=16 timeout 900 python -m pytest tests/test_gpu_local_ranks.py tests/test_gpu_single.py tests/test_gpu_row_blocks.py -q > $O/single_tests16.log 2>&1; echo "single16_rc=$?"; tail -15 $O/single_tests16.log
