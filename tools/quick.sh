# quick perf check: smoke + short bench with kernel diagnostics
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 120 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 300 python bench.py --no-extras --steps 20 --cpu-budget 0.2 --debug ${BENCH_ARGS} 2> gpurun_out/quick.err | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print('qps', round(r['value']), 'scan_ms', round(r['roofline']['scan_ms'],3), 'frac', round(r['roofline']['frac'],3), 'e2e', round(r['e2e']['value']), 'recall', r['recall_at_10'])"
grep -E "DEBUG|DENSE" gpurun_out/quick.err | cut -c1-400
