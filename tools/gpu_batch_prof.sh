cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 300 python tools/batch_prof.py 2
timeout -s KILL 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/batch_launches.csv python tools/batch_prof.py 2 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/batch_launches.csv
