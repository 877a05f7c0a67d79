#!/bin/bash
# build an alternative libpdx_b200 from a variant of one source file:
#   tools/ab_build.sh /tmp/pdx_batch_variant.cu pdx_batch.cu  ->  build_ab/libpdx_b200_alt.so
set -e
cd /root/repo/paper_2503_04422_b200/csrc
mkdir -p /root/repo/build_ab/obj
cp "$1" /root/repo/build_ab/obj/"$2"
for f in *.cuh; do cp $f /root/repo/build_ab/obj/; done
cd /root/repo/build_ab/obj
sed -i 's#"../../include/pdx_b200.h"#"/root/repo/include/pdx_b200.h"#' *.cuh *.cu 2>/dev/null || true
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O2 --cudart static -c -o alt.o "$2" 2>&1 | grep -E "error" || true
objs=$(ls /root/repo/paper_2503_04422_b200/csrc/*.o | grep -v "/${2%.cu}.o")
nvcc -gencode arch=compute_100a,code=sm_100a --cudart static -shared -o /root/repo/build_ab/libpdx_b200_alt.so alt.o $objs
echo "alt build ok"
