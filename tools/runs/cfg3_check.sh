mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_layer.py -x -q > gpurun_out/t_fused.log 2>&1; echo EXIT $? >> gpurun_out/t_fused.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
for c in cfg1 cfg3; do
timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/b_$c.json 2>/dev/null
SF_GEMM_LN_CLUSTER=1 timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/b_${c}_cl.json 2>/dev/null
done
tail -n 2 gpurun_out/t_fused.log; cat gpurun_out/smoke.log
for f in gpurun_out/b_cfg*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms']
print('$f', round(d['value']/1e6,2), 'e2e', round(d['e2e']['value']/1e6,2), [round(x/1e6,1) for x in d['e2e']['windows_tokens_per_s']], d['mha']['plan'], {a: round(b*1e3,1) for a,b in k.items()})"; done
