#!/bin/bash
# Build A/B variants of the library: scripts/build_variants.sh NAME "-DFOO=1 ..." ...
# (the flags go to both translation units; PTCFLAGS, default "-Xptxas -O1", to
# the tensor-core kernel's own)
cd /root/repo/paper_2406_03791_b200/csrc
PTCFLAGS=${PTCFLAGS--Xptxas -O1}
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  $NV $flags $PTCFLAGS -c -o /tmp/ptc_kernels_$name.o ptc_kernels.cu 2>&1 | grep -i error
  $NV $flags -shared -o ../librnntg_$name.so rnntg.cu /tmp/ptc_kernels_$name.o idle_trace.o -L/usr/local/cuda/lib64 -lcupti \
    -Xlinker -rpath=/usr/local/cuda/lib64 2>&1 | grep -i error
done
