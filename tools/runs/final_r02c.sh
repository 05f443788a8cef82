# round-2 final measurement set (one B200): tests, smoke, bench lines, launch list, ncu captures
mkdir -p gpurun_out/final3
O=gpurun_out/final3
timeout 1500 python -m pytest tests -m gpu -q > $O/gputest.log 2>&1; echo EXIT $? >> $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 900 python bench.py --impl reference > $O/bench_reference_cfg2.json 2> $O/bench_reference_cfg2.err
for c in cfg1 cfg3 cfg4; do timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_cfg2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"attn_tc|gemm2" -s 10 -c 5 -o $O/layer_cfg2 -f python tools/layer_once.py > $O/ncu_layer.log 2>&1
tail -n 2 $O/gputest.log; cat $O/smoke.log
timeout 900 python bench.py --sweep > $O/sweep_mha_v15.jsonl 2> $O/sweep.err
timeout 900 python bench.py --band-sweep --steps 7 > $O/band_sweep_v6.jsonl 2>/dev/null
