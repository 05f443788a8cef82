# A/B of the 64-row run boxes for consecutive column blocks (SF_ATTN_RUNBOX=0: one box per block)
for e in 1 0 1 0; do
SF_ATTN_RUNBOX=$e timeout 300 python tools/attn_cfg.py cfg2 | sed "s/^/runbox=$e /"
SF_ATTN_RUNBOX=$e timeout 600 python bench.py --no-cpu-baseline --steps 200 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('runbox=$e bench', round(d['value']/1e6,2), d['mha']['plan'], round(d['mha']['latency_us'],1))"
done
