cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for sp in 1 2 3 4 1 2; do
PDX_BATCH_SPLIT=$sp timeout 600 python bench.py --steps 30 --warmup 5 --no-extras > gpurun_out/bench_sp$sp.json 2> gpurun_out/bench_sp$sp.err
python -c "
import json
d=json.load(open('gpurun_out/bench_sp$sp.json'))
print('split', $sp, round(d['value']), d['ms_per_step'], round(d['e2e']['value']), round(d['roofline']['scan_ms'],4), d['parity']['ids_equal'])
"
done
