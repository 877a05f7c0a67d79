# batched pipeline debugging: per-phase syncs, hard timeouts
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export PDX_BATCH_DEBUG=1
timeout -s KILL 240 python -m pytest tests/test_gpu_batched.py -x -q -s --timeout 200 -k "bsa or small or dup" > gpurun_out/dbg_bsa.txt 2>&1; echo "bsa rc=$?"
grep -c "pdx batched" gpurun_out/dbg_bsa.txt; tail -n 12 gpurun_out/dbg_bsa.txt
timeout -s KILL 400 python bench.py --no-extras --steps 3 --warmup 3 --cpu-budget 0.2 --batched 2 > gpurun_out/dbg_bench.txt 2>&1; echo "bench rc=$?"
grep "pdx batched" gpurun_out/dbg_bench.txt | head -12; tail -n 3 gpurun_out/dbg_bench.txt | cut -c1-300
unset PDX_BATCH_DEBUG
timeout -s KILL 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_parity.py tests/test_handle.py -x -q --timeout 300 2>&1 | tail -n 6
for b in 1 2; do
timeout -s KILL 300 python bench.py --no-extras --steps 20 --cpu-budget 0.2 --batched $b 2>gpurun_out/b$b.err | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print('batched', $b, 'qps', round(r['value']), 'scan_ms', round(r['roofline']['scan_ms'],3), 'frac', round(r['roofline']['frac'],3), 'e2e', round(r['e2e']['value']), 'recall', r['recall_at_10'])"
done
