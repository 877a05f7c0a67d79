cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm --format=csv,noheader
timeout 900 python -m pytest tests/test_gpu_batched.py -x -q 2>&1 | tail -25 > gpurun_out/t1.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -8 >> gpurun_out/t1.txt
cat gpurun_out/t1.txt
for b in 1 2; do
timeout 300 python bench.py --no-extras --steps 20 --cpu-budget 0.2 --batched $b 2>gpurun_out/b$b.err | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print('batched', $b, 'qps', round(r['value']), 'scan_ms', round(r['roofline']['scan_ms'],3), 'frac', round(r['roofline']['frac'],3), 'e2e', round(r['e2e']['value']), 'recall', r['recall_at_10'])"
tail -3 gpurun_out/b$b.err
done
PDX_BATCH_DEBUG=1 timeout 300 python bench.py --no-extras --steps 3 --warmup 3 --cpu-budget 0.2 --batched 2 2>&1 >/dev/null | grep "pdx batched" | head -3
