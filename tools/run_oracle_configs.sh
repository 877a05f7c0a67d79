cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in c3 c4 c5; do
timeout 1500 python tools/oracle_configs.py $c > gpurun_out/oracle_$c.jsonl 2> gpurun_out/oracle_$c.err; echo $c=$?; cat gpurun_out/oracle_$c.jsonl; tail -3 gpurun_out/oracle_$c.err
done
free -g | head -2
