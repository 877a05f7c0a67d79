cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 300 python tools/phase1_diag.py 2>&1 | tail -n 8
timeout -s KILL 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:bscan_kernel -c 2 -o gpurun_out/bscan2 python tools/batch_prof.py 2 > gpurun_out/bscan_ncu.log 2>&1
tail -n 2 gpurun_out/bscan_ncu.log
