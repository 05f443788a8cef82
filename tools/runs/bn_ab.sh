# A/B of the selector's block_n widening (SF_PLAN_BN=0 keeps Eq. 2's block_n) on the bench configs
for c in cfg4 cfg2 cfg3 cfg1; do for e in 1 0; do
SF_PLAN_BN=$e timeout 600 python bench.py --config $c --no-cpu-baseline --steps 100 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$c bn=$e', round(d['value']/1e6,2), d['mha']['plan'], round(d['mha']['latency_us'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
