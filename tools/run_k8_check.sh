# K8 (tcgen05) checks on one B200: the tensor-core tests, then the C4 batch-1024 timing.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "tensor_core" > gpurun_out/t_k8.log 2>&1; echo k8tests=$?; tail -30 gpurun_out/t_k8.log
if [ -n "$FULL" ]; then
timeout 600 python -m pytest tests/test_handle.py -q -m gpu -x > gpurun_out/t_handle.log 2>&1; echo handle=$?; tail -3 gpurun_out/t_handle.log
fi
if [ -n "$C4" ]; then
timeout 900 python tools/k8_bench.py > gpurun_out/k8_bench.log 2>&1; echo k8bench=$?; tail -20 gpurun_out/k8_bench.log
fi
