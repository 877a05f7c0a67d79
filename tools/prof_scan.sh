mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-extras ${BENCH_ARGS}"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:pdx_scan_kernel -s 3 -c 1 -o gpurun_out/prof_scan -f $CMD > gpurun_out/ncu2.log 2>&1
echo ncu=$?
tail -1 gpurun_out/plain.log | cut -c1-300
