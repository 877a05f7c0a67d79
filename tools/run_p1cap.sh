cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for cap in 64 32 16 8; do for se in 64 256; do
PDX_P1CAP=$cap PDX_SURV_EXTRA=$se timeout 300 python bench.py --steps 30 --warmup 5 --no-extras --no-parity --cpu-budget 0.5 > gpurun_out/bcap.json 2>gpurun_out/bcap.err
python -c "import json;d=json.loads(open('gpurun_out/bcap.json').read().strip().splitlines()[-1]);p=d['roofline']['phases_ms_live'];print('cap $cap surv+$se', round(d['value']), round(d['ms_per_step'],4), {k:round(v*1000) for k,v in p.items()})"
PDX_BATCH_DEBUG=1 PDX_P1CAP=$cap PDX_SURV_EXTRA=$se timeout 300 python tools/one_search.py 2>&1 | grep "pdx batched" | tail -1
done; done
PDX_P1CAP=8 timeout 600 python -m pytest tests/test_gpu_c2.py tests/test_gpu_batched.py -q -m gpu -x > gpurun_out/t_cap.log 2>&1; echo tests_cap8=$?; tail -2 gpurun_out/t_cap.log
