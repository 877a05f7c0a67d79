# development loop for the MODE 0 head: batched/C2 tests, short bench, a full ncu capture of bscan MODE 0
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_c2.py -x -q --timeout 300 2>&1 | tail -n 3
timeout 600 python bench.py --steps 20 --warmup 5 --no-extras > gpurun_out/bench_apx.json 2> gpurun_out/bench_apx.err; echo bench=$?
python -c "
import json
d=json.load(open('gpurun_out/bench_apx.json'))
print(round(d['value']), d['ms_per_step'], round(d['e2e']['value']), {k: round(v*1000,1) for k,v in d['roofline']['phases_ms_live'].items()})
print(d['parity']['ids_equal'], d['parity']['dist_equal'])
"
if [ -n "$NCU" ]; then
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:bscan -c 1 -o gpurun_out/bscan_full -f python tools/one_search.py > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
fi
