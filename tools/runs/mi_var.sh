D=paper_2506_06095_b200
for v in "" mi4 mi5; do echo "== ${v:-default}"; if [ -n "$v" ]; then export SF_B200_LIB=$D/_lib_$v/libsf_b200.so; else unset SF_B200_LIB; fi
timeout 300 python tools/mi_sweep.py 2>&1 | head -3
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:mi_chain -s 2 -c 2 python tools/mi_once.py 2>&1 | grep -E "duration|dram__bytes" 
timeout 600 python bench.py --config cfg3 --no-cpu-baseline --steps 200 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms']
print('cfg3', round(d['value']/1e6,2), {a: round(b*1e3,1) for a,b in k.items() if 'mi' in a})"
done
