mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention.py -x -q -k "selector or dispatch" > gpurun_out/t_sel.log 2>&1; echo EXIT $? >> gpurun_out/t_sel.log
timeout 900 python bench.py --band-sweep --steps 7 > gpurun_out/band_sweep_v3.jsonl 2> gpurun_out/band_sweep.err
tail -n 3 gpurun_out/t_sel.log
python - <<'P'
import json
for l in open('gpurun_out/band_sweep_v3.jsonl'):
    d=json.loads(l); k='density' if 'density' in d else 'band'
    print(d['band_sweep'], d[k], d['reference_plan'], d['b200_plan'], round(d['blockwise_us'],1), round(d['rowwise_us'],1), round(d['regret_reference_mode'],2), round(d['regret_b200_mode'],2))
P
