mkdir -p gpurun_out
timeout 300 python tools/mi_sweep.py > gpurun_out/mi_sweep.txt 2>&1
timeout 300 ncu --set full --clock-control none -k regex:mi_chain -s 2 -c 1 -o gpurun_out/mi_ln -f python tools/mi_once.py > gpurun_out/ncu_mi.log 2>&1
cat gpurun_out/mi_sweep.txt; tail -3 gpurun_out/ncu_mi.log
