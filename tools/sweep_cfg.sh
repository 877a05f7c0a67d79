# Sweep scan CTA shapes (compute warps, tiles per claim, ring slots) on the bench workload.
mkdir -p gpurun_out
for w in ${WS:-8,4,32 4,4,16 4,2,8 4,2,16 2,4,8 2,2,4 2,2,8 3,4,16 1,4,4}; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-extras --warps $w --cpu-budget 0.2 ${BENCH_ARGS} > gpurun_out/sweep_$w.log 2>&1
  tail -1 gpurun_out/sweep_$w.log | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('$w', round(l['value']), round(l['roofline']['scan_ms'],3), round(l['roofline']['frac'],3), l['recall_at_10'])" 2>/dev/null || echo "$w failed"
done
