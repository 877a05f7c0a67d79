# Round measurement: GPU tests, default bench, ncu launch list + full capture of the scan kernel.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/gputest.log 2>&1; echo tests=$?; tail -3 gpurun_out/gputest.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench=$?; tail -1 gpurun_out/bench.log
CMD="python bench.py --steps 3 --warmup 3 --no-extras --cpu-budget 0.5"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:pdx_scan_kernel -s 3 -c 1 -o gpurun_out/prof_scan -f $CMD > gpurun_out/ncu2.log 2>&1
echo ncu=$?
