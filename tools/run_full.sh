# the round-end checks on one B200: the whole -m gpu suite, smoke, the default bench line,
# and (MULTI=1) a 2-rank gloo smoke run of bench.py's multi-GPU path on the one GPU
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/gputest_full.log 2>&1; echo tests=$?; tail -3 gpurun_out/gputest_full.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
if [ -n "$MULTI" ]; then
PDX_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_multi.json 2> gpurun_out/bench_multi.err; echo multi=$?; tail -c 800 gpurun_out/bench_multi.json; tail -5 gpurun_out/bench_multi.err
fi
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench=$?; tail -c 300 gpurun_out/bench_final.err
timeout 300 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?; cat gpurun_out/bench_ref.json | cut -c1-300
