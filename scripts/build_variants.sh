#!/bin/bash
# Build A/B variants of the library: scripts/build_variants.sh NAME "-DFOO=1 ..." ...
cd /root/repo/paper_2406_03791_b200/csrc
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr $flags -shared -o ../librnntg_$name.so rnntg.cu idle_trace.o -L/usr/local/cuda/lib64 -lcupti \
    -Xlinker -rpath=/usr/local/cuda/lib64 2>&1 | grep -i error
done
