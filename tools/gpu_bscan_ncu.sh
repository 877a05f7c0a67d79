cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:bscan_kernel -c 1 -o gpurun_out/bscan python tools/batch_prof.py 2 > gpurun_out/bscan_ncu.log 2>&1
tail -n 3 gpurun_out/bscan_ncu.log
python tools/ncu_summary.py gpurun_out/bscan.ncu-rep > gpurun_out/bscan_summary.txt 2>&1; head -n 70 gpurun_out/bscan_summary.txt
