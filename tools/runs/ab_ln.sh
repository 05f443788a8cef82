mkdir -p gpurun_out/ab
for i in 1 2; do for c in cfg2 cfg3 cfg4; do
timeout 900 python bench.py --config $c --no-cpu-baseline --steps 200 > gpurun_out/ab/p_${c}_$i.json 2>/dev/null
SF_GEMM_LN_CLUSTER=1 timeout 900 python bench.py --config $c --no-cpu-baseline --steps 200 > gpurun_out/ab/c_${c}_$i.json 2>/dev/null
done; done
for f in gpurun_out/ab/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms']
print('$f'.split('/')[-1], round(d['value']/1e6,2), 'us/step', round(d['ms_per_step']*1e3,1), {a: round(b*1e3,1) for a,b in k.items() if 'ln' in a})"; done
