#!/bin/bash
# Build A/B copies of libsdg_gpu.so with extra -D flags: variant_libs.sh name "-DFOO=1" ...
# Output: paper_2008_04356_b200/libsdg_gpu_<name>.so (select with SDG_GPU_LIB=...).
set -e
cd "$(dirname "$0")/../paper_2008_04356_b200/csrc"
ARCH="-gencode arch=compute_100a,code=sm_100a"
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden,-fvisibility-inlines-hidden --expt-relaxed-constexpr $flags -c kernels.cu -o /tmp/kernels_$name.o
  nvcc $ARCH -shared -cudart static -Xlinker --exclude-libs,ALL -o ../libsdg_gpu_$name.so build/host.o /tmp/kernels_$name.o build/solver.o -lnccl
  echo "built libsdg_gpu_$name.so ($flags)"
done
