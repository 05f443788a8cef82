# A/B of one-head (block_m 128) ring depths on cfg3/cfg4/dense shapes + the cfg4 bench
D=paper_2506_06095_b200
for v in "$@"; do echo "== ${v:-default}"; if [ -n "$v" ] && [ "$v" != default ]; then export SF_B200_LIB=$D/_lib_$v/libsf_b200.so; else unset SF_B200_LIB; fi
timeout 300 python tools/attn_cfg.py cfg3 cfg4 dense
timeout 600 python bench.py --config cfg4 --no-cpu-baseline --steps 100 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('cfg4 bench', round(d['value']/1e6,2), d['mha']['plan'], round(d['mha']['latency_us'],1), d['clocks']['sm_mhz'])"
done
