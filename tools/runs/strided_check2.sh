timeout 1500 python -m pytest tests/test_gpu_attention.py tests/test_gpu_layer.py tests/test_gpu_bench_shapes.py -q -x 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py --config cfg3 --no-cpu-baseline --steps 200 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms']
print('cfg3', round(d['value']/1e6,2), round(d['ms_per_step']*1e3,1), d['mha']['plan'], {a: round(b*1e3,1) for a,b in k.items()})"; done
timeout 900 python bench.py --sweep --patterns strided > gpurun_out/sweep_strided.jsonl 2>/dev/null
python -c "
import json
for l in open('gpurun_out/sweep_strided.jsonl'):
    d=json.loads(l); print(d['seq_len'], d['plan'], round(d['latency_us'],1), round(d['roofline']['frac'],3))"
