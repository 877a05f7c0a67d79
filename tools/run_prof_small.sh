cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/one_search.py > gpurun_out/one.log 2>&1 && \
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"select_warp|centroid_dist|project_kernel" -c 3 -o gpurun_out/small_full -f python tools/one_search.py > gpurun_out/ncu3.log 2>&1; echo ncu=$?
