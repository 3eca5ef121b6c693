cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_local_ranks.py -q -x -k "more_ranks" > $O/edge.log 2>&1; echo "edge_rc=$?"; tail -30 $O/edge.log
for v in 9 16 17 18 9 16; do IPT_SPMV_VARIANT=$v timeout 300 python tools/spmv_probe.py 2>&1 | tail -1; done
