#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out
./tools/cpp/api_latency 1024 2>&1 | tail -3
./tools/cpp/api_latency 256 2>&1 | tail -1
timeout 1200 python bench.py > $O/bench_r01b.json 2> $O/bench_r01b.err; echo "bench_rc=$?"; cat $O/bench_r01b.json | head -c 6000; tail -3 $O/bench_r01b.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref_rc=$?"; cat $O/bench_ref.json
