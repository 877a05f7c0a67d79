cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python tools/oracle_configs.py c4 > gpurun_out/oracle_c4.jsonl 2> gpurun_out/oracle_c4.err; echo c4=$?; cat gpurun_out/oracle_c4.jsonl; tail -3 gpurun_out/oracle_c4.err
for dn in 0 1; do
PDX_BSCAN_DENSE=$dn timeout 300 python bench.py --steps 30 --warmup 5 --no-extras --no-parity --cpu-budget 0.5 > gpurun_out/bdense$dn.json 2>gpurun_out/bdense$dn.err; echo dense=$dn rc=$?
python -c "import json;d=json.loads(open('gpurun_out/bdense$dn.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['roofline']['phases_ms_live'])"
done
PDX_BSCAN_DENSE=1 timeout 600 python -m pytest tests/test_gpu_c2.py tests/test_gpu_batched.py -q -m gpu -x > gpurun_out/t_dense.log 2>&1; echo tests_dense=$?; tail -2 gpurun_out/t_dense.log
