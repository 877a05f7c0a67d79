cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"bscan_kernel|bchain1|bdense" -c 5 -o gpurun_out/p4 python tools/batch_prof.py 2 > gpurun_out/p4.log 2>&1
tail -n 1 gpurun_out/p4.log
