mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/gputest.log 2>&1; echo tests=$?; tail -2 gpurun_out/gputest.log
for w in ${WS:-6,2,12}; do timeout 300 python bench.py --steps 5 --warmup 3 --no-extras --warps $w --cpu-budget 0.5 --debug > gpurun_out/bench_w$w.log 2> gpurun_out/bench_w$w.err; grep DEBUG gpurun_out/bench_w$w.err; tail -1 gpurun_out/bench_w$w.log | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('$w', round(l['value']), round(l['roofline']['scan_ms'],3), round(l['roofline']['frac'],3), l['recall_at_10'])"; done
