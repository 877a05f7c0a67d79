cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python tools/bench_configs.py c3 > gpurun_out/configs_c3.jsonl 2> gpurun_out/configs_c3.err; echo c3=$?; cut -c1-300 gpurun_out/configs_c3.jsonl
timeout 1500 python tools/c5_sharded.py --emulate-rank 0 --world 8 > gpurun_out/c5_rank0.jsonl 2> gpurun_out/c5_rank0.err; echo c5=$?; cut -c1-400 gpurun_out/c5_rank0.jsonl; tail -2 gpurun_out/c5_rank0.err
timeout 1500 python tools/oracle_configs.py c3 > gpurun_out/oracle_c3b.jsonl 2> gpurun_out/oracle_c3b.err; echo oc3=$?; cat gpurun_out/oracle_c3b.jsonl
