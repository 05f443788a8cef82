# A/B of the head-pair 5-D K/V boxes (SF_ATTN_PAIR5=0: one box per head) at the cfg2 plan (64,16)
for e in 1 0 1 0; do
SF_ATTN_PAIR5=$e timeout 600 python bench.py --no-cpu-baseline --steps 200 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms']
print('cfg2 pair5=$e', round(d['value']/1e6,2), d['mha']['plan'], round(d['mha']['latency_us'],1))"
done
