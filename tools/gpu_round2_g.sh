cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_local_ranks.py -q -x -k batch > $O/batch.log 2>&1; echo "batch_rc=$?"; tail -3 $O/batch.log
timeout 600 ./oracle/_ref/acceptance_b200 2>&1 | grep -i "criterion 9\|criteria"
IPT_PROFILE=1 timeout 300 python tools/profile_config5_e2e.py 2>&1 | tail -8
python bench.py --gpus 2 --steps 1; echo "bench_gpus2_rc=$?"
timeout 900 python tools/sanitize_smoke.py > $O/sanitize_plain.log 2>&1; echo "plain_rc=$?"; tail -2 $O/sanitize_plain.log
timeout 1800 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_smoke.py > $O/memcheck.log 2>&1; echo "memcheck_rc=$?"; tail -6 $O/memcheck.log
