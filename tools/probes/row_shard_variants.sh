for v in 16 12 13 9 7 18; do echo "variant $v"; IPT_SPMV_VARIANT=$v timeout 300 python tools/row_shard_probe.py 2>&1 | grep -E '"gpus": (1|8)' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['gpus'], round(d['rank_step_ms'],4))
"; done
