for e in 1 0 1 0; do SF_PLAN_PAIR=0 SF_ATTN_RUNBOX=$e timeout 300 python tools/attn_cfg.py cfg2 cfg3 cfg4 dense | sed "s/^/runbox=$e bm128 /"; done
for e in 1 0; do SF_ATTN_RUNBOX=$e timeout 600 python bench.py --config cfg3 --no-cpu-baseline --steps 100 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('runbox=$e cfg3', round(d['value']/1e6,2), d['mha']['plan'], round(d['mha']['latency_us'],1))"; done
