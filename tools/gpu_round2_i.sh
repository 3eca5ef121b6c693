cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_single.py tests/test_gpu_local_ranks.py tests/test_gpu_row_blocks.py -q -x > $O/single.log 2>&1; echo "single_rc=$?"; tail -3 $O/single.log
IPT_PROFILE=1 timeout 300 python tools/profile_config5_e2e.py 2>&1 | tail -5
timeout 900 python bench.py --steps 2 --warmup 3 --secondary none --no-e2e --no-cpu > $O/bench_small.json 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_r02.csv python bench.py --steps 2 --warmup 3 --secondary none --no-e2e --no-cpu > $O/ncu_launch.log 2>&1; echo "ncu_rc=$?"
