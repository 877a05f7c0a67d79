cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 240 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "tensor_core and not auto" > gpurun_out/t_k8pair.log 2>&1; echo k8tests=$?; tail -25 gpurun_out/t_k8pair.log
if grep -q passed gpurun_out/t_k8pair.log && ! grep -q failed gpurun_out/t_k8pair.log; then
K8_PRECISION=tf32 timeout -s KILL 600 python tools/k8_bench.py > gpurun_out/k8_bench.log 2>&1; echo k8bench=$?; tail -4 gpurun_out/k8_bench.log | cut -c1-420
PDX_K8_PAIR=0 K8_PRECISION=tf32 timeout -s KILL 600 python tools/k8_bench.py > gpurun_out/k8_bench1.log 2>&1; echo k8bench1=$?; tail -4 gpurun_out/k8_bench1.log | cut -c1-420
fi
