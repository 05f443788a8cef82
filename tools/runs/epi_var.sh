D=paper_2506_06095_b200
SF_B200_LIB=$D/_lib_epi16/libsf_b200.so timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_layer.py -q -x 2>&1 | tail -2
for v in "" epi16; do echo "== ${v:-default}"; if [ -n "$v" ]; then export SF_B200_LIB=$D/_lib_$v/libsf_b200.so; else unset SF_B200_LIB; fi
timeout 300 python tools/ln_time.py 2>&1 | head -2
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --steps 200 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms']
print('cfg2', round(d['value']/1e6,2), {a: round(b*1e3,1) for a,b in k.items() if 'ln' in a})"; done
done
