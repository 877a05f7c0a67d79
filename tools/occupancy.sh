# per-query scan time vs resident query CTAs per SM (nq = 148 k)
cd $GRAFT_REPO_ROOT
for nq in 148 296 444 592 888; do
  python bench.py --nq $nq --steps 20 --no-extras --cpu-budget 0.1 --debug 2>gpurun_out/occ.err | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print($nq, 'qps', round(r['value']), 'scan_ms', round(r['roofline']['scan_ms'],3))"
  grep DEBUG gpurun_out/occ.err | cut -c1-120
done
