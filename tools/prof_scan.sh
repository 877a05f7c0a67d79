mkdir -p gpurun_out
set -x
for w in 4 8 16; do timeout 300 python bench.py --steps 5 --warmup 3 --no-extras --warps $w > gpurun_out/bench_w$w.log 2>&1; tail -1 gpurun_out/bench_w$w.log | python -c "import json,sys; l=json.loads(sys.stdin.read()); print($w, l['value'], l['roofline']['scan_ms'], l['roofline']['frac'])"; done
CMD="python bench.py --steps 3 --warmup 3 --no-extras"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:pdx_scan_kernel -s 3 -c 1 -o gpurun_out/prof_scan $CMD > gpurun_out/ncu2.log 2>&1
echo ncu=$?
