cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out; mkdir -p $O
for v in 16 19 20 21 16 19 21; do IPT_SPMV_VARIANT=$v timeout 300 python tools/spmv_probe.py 2>&1 | tail -1; done
IPT_SPMV_VARIANT=19 timeout 900 python -m pytest tests/test_gpu_single.py tests/test_gpu_row_blocks.py tests/test_gpu_local_ranks.py -q -x -k "csr or CSR or row" > $O/v19.log 2>&1; echo "v19_rc=$?"; tail -3 $O/v19.log
