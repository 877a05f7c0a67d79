cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/one_search.py > gpurun_out/one.log 2>&1 && \
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,launch__registers_per_thread --clock-control none --csv --log-file gpurun_out/search_kernels.csv python tools/one_search.py > gpurun_out/ncu1.log 2>&1; echo ncu1=$?
