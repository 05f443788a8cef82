mkdir -p gpurun_out
for m in bigbird dense; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_tc -s 1 -c 1 -o gpurun_out/attn3b_$m -f python tools/attn_once.py $m 16 > gpurun_out/ncu_attn3b_$m.log 2>&1
done
