cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_c2.py tests/test_gpu_batched.py -q -m gpu -x > gpurun_out/t_perf.log 2>&1; echo tests=$?; tail -2 gpurun_out/t_perf.log
for v in 0 1; do
if [ $v = 1 ]; then export PDX_NO_QPERM=1; fi
timeout 300 python bench.py --steps 30 --warmup 5 --no-extras --no-parity --cpu-budget 0.5 > gpurun_out/bperf$v.json 2>gpurun_out/bperf$v.err; echo bench=$?
python -c "import json;d=json.loads(open('gpurun_out/bperf$v.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['e2e']['value']);print(d['roofline']['phases_ms_live'])"
done
unset PDX_NO_QPERM
timeout 300 python tools/one_search.py > gpurun_out/one.log 2>&1 && \
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,launch__registers_per_thread --clock-control none --csv --log-file gpurun_out/search_kernels.csv python tools/one_search.py > gpurun_out/ncu1.log 2>&1; echo ncu1=$?
