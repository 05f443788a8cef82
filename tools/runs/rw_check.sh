mkdir -p gpurun_out
timeout 300 python tools/rw_time.py > gpurun_out/rw_time.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:rowwise -s 1 -c 1 -o gpurun_out/rw_band1 -f python tools/rw_once.py 1 2048 > gpurun_out/ncu_rw.log 2>&1
cat gpurun_out/rw_time.txt
