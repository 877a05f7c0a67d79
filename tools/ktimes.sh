# per-kernel device time of one C2 search (ncu launch list)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/one_search.py > gpurun_out/ncu1.log 2>&1; echo ncu=$?
python tools/launch_table.py gpurun_out/launches.csv
