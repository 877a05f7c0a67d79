cd $GRAFT_REPO_ROOT
for v in "1 1 0" "0 0 0"; do
  set -- $v
  make -C paper_2503_04422_b200/csrc clean >/dev/null; make -C paper_2503_04422_b200/csrc -j8 NVFLAGS="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O2 --cudart static -DPDX_MBAR_RING=$1 -DPDX_MBAR_COMMIT=$2 -DPDX_MBAR_HINT=$3" >/dev/null 2>&1
  timeout 60 python __graft_entry__.py smoke > gpurun_out/smoke_$1$2$3.log 2>&1; echo "ring=$1 commit=$2 hint=$3 smoke=$?"; tail -1 gpurun_out/smoke_$1$2$3.log | cut -c1-200
  timeout 300 python bench.py --no-extras --steps 20 --cpu-budget 0.2 --debug 2> gpurun_out/bench_$1$2$3.err | cut -c1-240; grep DEBUG gpurun_out/bench_$1$2$3.err
done
