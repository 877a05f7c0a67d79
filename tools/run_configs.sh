cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python tools/bench_configs.py c1 c3 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo configs=$?; cut -c1-330 gpurun_out/configs.jsonl; tail -3 gpurun_out/configs.err
timeout 1500 python tools/oracle_configs.py c5 > gpurun_out/oracle_c5b.jsonl 2> gpurun_out/oracle_c5b.err; echo c5=$?; cat gpurun_out/oracle_c5b.jsonl; tail -3 gpurun_out/oracle_c5b.err
