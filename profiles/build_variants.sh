#!/bin/bash
# Build libgconn variants that differ in one uf_kernels.cu compile-time tuning
# (A/B on the GPU box with GC_LIB_VARIANT=<name>); usage: build_variants.sh name:"-DFLAG=.." ...
set -e
cd "$(dirname "$0")/.."
P=paper_2008_11839_b200
mkdir -p $P/_variants /tmp/gcvar
objs=$(ls $P/_build_obj/*.o | grep -v uf_kernels.o)
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC \
    -I include $flags -c $P/csrc/uf_kernels.cu -o /tmp/gcvar/uf_$name.o &
done
wait
for spec in "$@"; do
  name=${spec%%:*}
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $P/_variants/libgconn_$name.so $objs /tmp/gcvar/uf_$name.o -lcudart_static -ldl
done
ls -la $P/_variants
