timeout 1200 python -m pytest tests/test_gpu_fused.py tests/test_gpu_layer.py tests/test_gpu_bench_shapes.py -q -x 2>&1 | tail -2
for c in cfg1 cfg2 cfg3 cfg4; do timeout 600 python bench.py --config $c --no-cpu-baseline --steps 200 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$c', round(d['value']/1e6,2), round(d['ms_per_step']*1e3,1))"; done
