# scan occupancy experiment: rebuild with PDX_SCAN_MIN_BLOCKS=$MB and sweep CTA shapes
cd $GRAFT_REPO_ROOT
make -C paper_2503_04422_b200/csrc clean >/dev/null
make -C paper_2503_04422_b200/csrc -j8 NVFLAGS="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O2 --cudart static -Xptxas -warn-spills -DPDX_SCAN_MIN_BLOCKS=$MB" 2>&1 | grep -i "spill" | grep "ILi8ELb0ELi0" | head -2
timeout 120 python __graft_entry__.py smoke 2>&1 | tail -1
bash tools/sweep_cfg.sh
