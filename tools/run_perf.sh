# correctness of the batched pipeline (C2 vs the reference golden + oracle, batched vs per-query
# scan and oracle) then the C2 bench line (phases)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_c2.py tests/test_gpu_batched.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/t_perf.log 2>&1; echo tests=$?; tail -2 gpurun_out/t_perf.log
timeout 300 python bench.py --steps 30 --warmup 5 --no-extras --no-parity --cpu-budget 0.5 > gpurun_out/bperf.json 2>gpurun_out/bperf.err; echo bench=$?
python -c "import json;d=json.loads(open('gpurun_out/bperf.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['e2e']['value']);print(d['roofline']['phases_ms_live'])"
