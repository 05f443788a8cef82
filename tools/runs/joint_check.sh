timeout 900 python -m pytest tests/test_gpu_fused.py -q -x -k "layernorm or large or ln" 2>&1 | tail -2
timeout 300 python tools/ln_time.py
SF_B200_LIB=paper_2506_06095_b200/_lib_trace/libsf_b200.so timeout 300 python tools/gemm_ln_trace.py 2>&1 | tail -6
