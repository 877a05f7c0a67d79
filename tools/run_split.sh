cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
PDX_BATCH_SPLIT=2 timeout 600 python -m pytest tests/test_gpu_c2.py tests/test_gpu_batched.py -q -m gpu -x > gpurun_out/t_split.log 2>&1; echo tests_split2=$?; tail -2 gpurun_out/t_split.log
for sp in 1 2 3 4; do
PDX_BATCH_SPLIT=$sp timeout 300 python bench.py --steps 30 --warmup 5 --no-extras --no-parity --cpu-budget 0.5 > gpurun_out/bsplit$sp.json 2>gpurun_out/bsplit$sp.err; echo split=$sp rc=$?
python -c "import json;d=json.loads(open('gpurun_out/bsplit$sp.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['e2e']['value'])"
done
