#!/bin/bash
# Build A/B variants of the library: scripts/build_variants.sh NAME "-DFOO=1 ..." ...
# The flags go to the tensor-core kernel's translation unit (ptc_kernels.cu,
# PTCFLAGS default "-Xptxas -O1"); rnntg.cu is compiled once (RNNTG_FLAGS).
set -e
cd /root/repo/paper_2406_03791_b200/csrc
PTCFLAGS=${PTCFLAGS--Xptxas -O1}
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
$NV $RNNTG_FLAGS -c -o /tmp/rnntg_host_variant.o rnntg.cu
pids=()
args=("$@")
for ((i = 0; i < ${#args[@]}; i += 2)); do
  name=${args[i]}; flags=${args[i+1]}
  ( $NV $flags $PTCFLAGS -c -o /tmp/ptc_kernels_$name.o ptc_kernels.cu && \
    $NV -shared -o ../librnntg_$name.so /tmp/rnntg_host_variant.o /tmp/ptc_kernels_$name.o idle_trace.o \
      -L/usr/local/cuda/lib64 -lcupti -Xlinker -rpath=/usr/local/cuda/lib64 ) &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
