# full ncu capture of one kernel (regex $K) of one C2 search; env passes through
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:$K -c 1 -o gpurun_out/kern_$K -f python tools/one_search.py > gpurun_out/ncu_$K.log 2>&1; echo ncu=$?
