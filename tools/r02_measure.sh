# Round-2 measurement on one B200: GPU tests, smoke, default bench line, ncu
# per-launch metrics of one C2 search (tools/one_search.py), a full capture
# of bscan MODE 0.  Then, here: python tools/ncu_kernels.py
#   gpurun_out/search_kernels.csv profiles/r02_kernels.json
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=${TESTS:-tests}
timeout 1200 python -m pytest $T -q -m gpu -x > gpurun_out/gputest.log 2>&1; echo tests=$?; tail -3 gpurun_out/gputest.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?; tail -c 600 gpurun_out/bench.err
if [ -n "$NCU" ]; then
# (ncu serialises kernels: the phase-1 chain kernel must not wait for a dense kernel that
# cannot run next to it — PDX_P1_OVERLAP=0 launches the two one after the other)
export PDX_P1_OVERLAP=0
timeout 300 python tools/one_search.py > gpurun_out/one.log 2>&1 && \
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,launch__registers_per_thread --clock-control none --csv --log-file gpurun_out/search_kernels.csv python tools/one_search.py > gpurun_out/ncu1.log 2>&1; echo ncu1=$?
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:bscan0_kernel -c 1 -o gpurun_out/bscan_full -f python tools/one_search.py > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
fi
