cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "select_buckets" > gpurun_out/t_sel.log 2>&1; echo tests=$?; tail -3 gpurun_out/t_sel.log
timeout 1500 python tools/c5_sharded.py --emulate-rank 0 --world 8 > gpurun_out/c5_rank0.jsonl 2> gpurun_out/c5_rank0.err; echo c5=$?; cat gpurun_out/c5_rank0.jsonl; tail -3 gpurun_out/c5_rank0.err
