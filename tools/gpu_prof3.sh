cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"bscan_kernel|bchain1" -c 3 -o gpurun_out/bscan3 python tools/batch_prof.py 2 > gpurun_out/bscan_ncu.log 2>&1
tail -n 2 gpurun_out/bscan_ncu.log
