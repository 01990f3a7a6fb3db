#!/bin/bash
# Ablation builds of the E4M3 screen for profiles/r02_screen_ablation.md (timing
# only, labels meaningless): PCB_ABL=1 drops the epilogue's arithmetic (keeps its
# TMEM loads and handshakes), PCB_ABL=2 also drops the TMEM loads.  The hooks are
# applied to a temporary copy of the kernel; the libraries go to build_exp/
# (git-ignored), then run scripts/gpu_abl.sh under gpurun.
set -e
cd "$(dirname "$0")/.."
mkdir -p build_exp
python - <<'PY'
s = open("paper_2501_05587_b200/csrc/assign_screen_bf16.cu").read()
s = s.replace("""          if (CAND) {
            sb_chunk_cand(cur0, c0 + 32 * qa, thr, row, n, rc, cand, nc);""", """#if defined(PCB_ABL)
          if (!CAND) { R1 = fminf(R1, __uint_as_float(cur0[0] ^ cur1[5])); } else
#endif
          if (CAND) {
            sb_chunk_cand(cur0, c0 + 32 * qa, thr, row, n, rc, cand, nc);""")
import re
s = re.sub(r"(\n(\s*)ptx::tmem_ld_32x32b_x32_async\([^\n]*\n\s*ptx::tmem_ld_32x32b_x32_async\([^\n]*)",
           r"\n#if !defined(PCB_ABL) || PCB_ABL < 2\1\n#endif", s)
open("build_exp/assign_screen_bf16_abl.cu", "w").write(s)
PY
for a in 1 2; do
  nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr \
       -DPCB_ABL=$a -Ipaper_2501_05587_b200/csrc -c build_exp/assign_screen_bf16_abl.cu -o build_exp/asb_abl$a.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -Xcompiler -pthread \
       -o build_exp/libabl$a.so $(ls build/*.o | grep -v assign_screen_bf16.o) build_exp/asb_abl$a.o
done
