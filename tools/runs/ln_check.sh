mkdir -p gpurun_out
timeout 300 python tools/ln_time.py > gpurun_out/ln_time.txt 2>&1
SF_B200_LIB=paper_2506_06095_b200/_lib_trace/libsf_b200.so timeout 300 python tools/gemm_ln_trace.py > gpurun_out/ln_trace.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_layer.py -x -q > gpurun_out/t_fused.log 2>&1; echo EXIT $? >> gpurun_out/t_fused.log
tail -n 3 gpurun_out/t_fused.log; cat gpurun_out/ln_time.txt gpurun_out/ln_trace.txt
