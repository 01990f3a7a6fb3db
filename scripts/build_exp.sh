#!/bin/bash
# Build experiment variants of the library into build_exp/lib<tag>.so:
#   scripts/build_exp.sh <tag> <extra nvcc flags...>
set -e
tag=$1; shift
mkdir -p build_exp/$tag
for f in paper_2501_05587_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr "$@" -c $f -o build_exp/$tag/$b.o &
done
for f in paper_2501_05587_b200/csrc/*.cpp; do
  g++ -O3 -std=c++17 -fPIC -pthread -c $f -o build_exp/$tag/$(basename $f .cpp).cpp.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -Xcompiler -pthread -o build_exp/lib$tag.so build_exp/$tag/*.o
echo built build_exp/lib$tag.so
