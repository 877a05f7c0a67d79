# iterate: batched + parity tests, bench both modes, launch table of one batched search
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_parity.py tests/test_handle.py -x -q --timeout 300 2>&1 | tail -n 8
for b in ${MODES:-2}; do
timeout -s KILL 300 python bench.py --no-extras --steps 20 --cpu-budget 0.2 --batched $b 2>gpurun_out/b$b.err | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print('batched', $b, 'qps', round(r['value']), 'scan_ms', round(r['roofline']['scan_ms'],3), 'frac', round(r['roofline']['frac'],3), 'e2e', round(r['e2e']['value']), 'recall', r['recall_at_10'])"
done
PDX_BATCH_DEBUG=1 timeout -s KILL 300 python tools/batch_prof.py 2 2>&1 | tail -n 2
timeout -s KILL 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/batch_launches.csv python tools/batch_prof.py 2 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/batch_launches.csv
