mkdir -p gpurun_out
timeout 300 python tools/attn_cfg.py cfg2 cfg3 cfg4 dense > gpurun_out/attn_cfg_v3.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_attention.py -x -q > gpurun_out/t_attn.log 2>&1; echo EXIT $? >> gpurun_out/t_attn.log
timeout 900 python -m pytest tests/test_gpu_bench_shapes.py -x -q -k "mha" > gpurun_out/t_shapes.log 2>&1; echo EXIT $? >> gpurun_out/t_shapes.log
tail -n 3 gpurun_out/t_attn.log gpurun_out/t_shapes.log; cat gpurun_out/attn_cfg_v3*.txt
