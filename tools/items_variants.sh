# sparse-phase capacity experiment: PDX_ITEMS_PER_WARP in {32, 48, 64, 96}
cd $GRAFT_REPO_ROOT
for ipw in 32 48 64 96; do
  make -C paper_2503_04422_b200/csrc clean >/dev/null
  make -C paper_2503_04422_b200/csrc -j8 NVFLAGS="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O2 --cudart static -DPDX_ITEMS_PER_WARP=$ipw" >/dev/null 2>&1
  echo "items/warp $ipw: $(timeout 120 python __graft_entry__.py smoke 2>&1 | tail -1 | cut -c1-30)"
  WS="8,4,32" bash tools/sweep_cfg.sh
done
