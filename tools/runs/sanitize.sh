mkdir -p gpurun_out/san
timeout 300 python tools/sanitize_once.py > gpurun_out/san/plain.txt 2>&1
for t in racecheck synccheck memcheck; do
timeout 1500 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_once.py > gpurun_out/san/$t.txt 2>&1
done
tail -n 4 gpurun_out/san/*.txt
