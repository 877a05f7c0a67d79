# diagnostics build: per-phase cycle counters compiled in, then a --debug bench
cd $GRAFT_REPO_ROOT
make -C paper_2503_04422_b200/csrc clean >/dev/null
make -C paper_2503_04422_b200/csrc -j8 NVFLAGS="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O2 --cudart static -DPDX_SCAN_PROFILE=1 ${EXTRA_NVFLAGS}" >/dev/null 2>&1
bash tools/quick.sh
