cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
K8_PROF=1 timeout 300 python tools/k8_bench.py > gpurun_out/k8p_plain.log 2>&1 && \
K8_PROF=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k8_tc_kernel -s 1 -c 1 -o gpurun_out/k8_full -f python tools/k8_bench.py > gpurun_out/k8p_ncu.log 2>&1; echo ncu=$?
K8_PROF=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/k8_launches.csv python tools/k8_bench.py > gpurun_out/k8p_ncu2.log 2>&1; echo ncu2=$?
