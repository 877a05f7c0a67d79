mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/gputest.log 2>&1; echo tests=$?; tail -3 gpurun_out/gputest.log
for w in ${WS:-2,2 4,1 4,2 4,4 8,1 8,2}; do timeout 300 python bench.py --steps 5 --warmup 3 --no-extras --warps $w --cpu-budget 0.5 > gpurun_out/bench_w$w.log 2>&1; tail -1 gpurun_out/bench_w$w.log | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('$w', round(l['value']), round(l['roofline']['scan_ms'],3), round(l['roofline']['frac'],3), l['recall_at_10'])"; done
