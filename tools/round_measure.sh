# Round measurement: GPU tests, smoke, default bench, ncu launch list (+ DRAM) of one
# batched search and a full capture of its dominant kernel.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/gputest.log 2>&1; echo tests=$?; tail -3 gpurun_out/gputest.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 300 python tools/batch_prof.py 0 > gpurun_out/plain.log 2>&1; echo plain=$?; tail -1 gpurun_out/plain.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/search_metrics.csv python tools/batch_prof.py 0 > gpurun_out/ncu1.log 2>&1; echo ncu1=$?
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:bscan_kernel -c 1 -o gpurun_out/bscan_full -f python tools/batch_prof.py 0 > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
# then, here: python tools/batch_report.py r01 gpurun_out/search_metrics.csv gpurun_out/bscan_full.ncu-rep
# (writes profiles/, which bench.py reads), and a second call: python bench.py
