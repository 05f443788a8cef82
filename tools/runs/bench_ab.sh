mkdir -p gpurun_out
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --steps 200 > gpurun_out/bench_new_$i.json 2>/dev/null
SF_GEMM_LN_CLUSTER=1 timeout 600 python bench.py --no-cpu-baseline --steps 200 > gpurun_out/bench_old_$i.json 2>/dev/null
done
for f in gpurun_out/bench_new_*.json gpurun_out/bench_old_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms']
print('$f', round(d['value']/1e6,2), 'e2e', round(d['e2e']['value']/1e6,2), {a: round(b*1e3,1) for a,b in k.items()})"; done
