# A/B on one box: the in-tree library vs build_ab/libpdx_b200_alt.so, interleaved
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in 1 2; do
for v in A B; do
if [ $v = B ]; then export PDX_B200_LIB=$GRAFT_REPO_ROOT/build_ab/libpdx_b200_alt.so; else unset PDX_B200_LIB; fi
timeout 600 python bench.py --steps 30 --warmup 5 --no-extras > gpurun_out/bench_$v$i.json 2> gpurun_out/bench_$v$i.err
python -c "
import json
d=json.load(open('gpurun_out/bench_$v$i.json'))
print('$v', round(d['value']), d['ms_per_step'], round(d['e2e']['value']), round(d['roofline']['scan_ms'],4), d['parity']['ids_equal'])
"
done; done
