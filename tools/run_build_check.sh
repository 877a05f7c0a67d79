cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_build.py tests/test_handle.py -q -m gpu > gpurun_out/t_build.log 2>&1; echo tests=$?; tail -25 gpurun_out/t_build.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-parity > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo bench=$?; tail -c 1500 gpurun_out/bench2.err
