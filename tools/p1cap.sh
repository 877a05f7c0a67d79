cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in 64 48 40 32 64 48; do
PDX_P1CAP=$c timeout 600 python bench.py --steps 20 --warmup 5 --no-extras > gpurun_out/bench_cap$c.json 2> gpurun_out/bench_cap$c.err
python -c "
import json
d=json.load(open('gpurun_out/bench_cap$c.json'))
print($c, round(d['value']), d['ms_per_step'], round(d['e2e']['value']), {k: round(v*1000,1) for k,v in d['roofline']['phases_ms_live'].items()}, d['parity']['ids_equal'])
"
done
