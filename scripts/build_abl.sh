#!/bin/bash
# Ablation builds of the E4M3 screen for profiles/r02_screen_ablation.md (timing
# only, labels meaningless): PCB_ABL=1 drops the epilogue's arithmetic, 2 also its
# TMEM loads.  The PCB_ABL hooks are not kept in the tree: apply them to a copy
# (see the profile for the two edits) and build into build_exp/libabl<n>.so, then
# run scripts/gpu_abl.sh under gpurun.
set -e
cd "$(dirname "$0")/.."
src=${1:-paper_2501_05587_b200/csrc/assign_screen_bf16.cu}
mkdir -p build_exp
for a in 1 2; do
  nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr \
       -DPCB_ABL=$a -Ipaper_2501_05587_b200/csrc -c "$src" -o build_exp/asb_abl$a.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -Xcompiler -pthread \
       -o build_exp/libabl$a.so $(ls build/*.o | grep -v assign_screen_bf16.o) build_exp/asb_abl$a.o
done
