mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fused.py -x -q -k chain > gpurun_out/t_cici.log 2>&1; echo EXIT $? >> gpurun_out/t_cici.log
timeout 900 python -m pytest tests/test_cpp_host_api.py -x -q > gpurun_out/t_cpp.log 2>&1; echo EXIT $? >> gpurun_out/t_cpp.log
tail -n 3 gpurun_out/t_cici.log gpurun_out/t_cpp.log
