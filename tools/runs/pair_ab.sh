# A/B of the selector's head-pair choice (SF_PLAN_PAIR=0 keeps block_m 128) on the bench configs
for c in cfg2 cfg1 cfg3 cfg4; do for e in 1 0 1 0; do
SF_PLAN_PAIR=$e timeout 600 python bench.py --config $c --no-cpu-baseline --steps 200 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms']
print('$c pair=$e', round(d['value']/1e6,2), d['mha']['plan'], round(d['mha']['latency_us'],1), 'e2e', round(d['e2e']['value']/1e6,2))"
done; done
