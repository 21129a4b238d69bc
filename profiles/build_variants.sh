#!/bin/bash
# Build libgconn variants that differ in one source file's compile-time tuning
# (A/B on the GPU box with GC_LIB_VARIANT=<name>).
#   build_variants.sh name:file.cu:"-DFLAG=.." ...   (file relative to csrc/)
set -e
cd "$(dirname "$0")/.."
P=paper_2008_11839_b200
mkdir -p $P/_variants /tmp/gcvar
for spec in "$@"; do
  IFS=: read -r name file flags <<< "$spec"
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC \
    -I include $flags -c $P/csrc/$file -o /tmp/gcvar/${name}.o &
done
wait
for spec in "$@"; do
  IFS=: read -r name file flags <<< "$spec"
  objs=$(ls $P/_build_obj/*.o | grep -v "/${file%.cu}.o")
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $P/_variants/libgconn_$name.so $objs /tmp/gcvar/${name}.o -lcudart_static -ldl
done
ls -la $P/_variants
