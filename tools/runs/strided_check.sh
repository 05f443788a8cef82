timeout 900 python -m pytest tests/test_gpu_attention.py -q -x -k strided 2>&1 | tail -3
timeout 600 python tools/strided_time.py
