// Microbenchmark: tcgen05.ld (LDTM) throughput per SM on one B200, by shape and
// packing — how many TMEM columns x lanes per clock an epilogue can read.
// One CTA per SM (all 148), W warps, each warp loops over its 32-lane slice of
// a 512-column allocation issuing two loads per wait.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a scripts/tmem_ld_probe.cu -o build/tmem_ld_probe
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2501_05587_b200/csrc/tc_ptx.cuh"

using namespace pcb;

#define LD32(shape, taddr, r)                                                                              \
  asm volatile("tcgen05.ld.sync.aligned." shape ".b32 "                                                   \
               "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"                                  \
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),      \
                 "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),  \
                 "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),            \
                 "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),            \
                 "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])             \
               : "r"(taddr))

// MODE 0: 32x32b.x32 (32 columns per load); 1: 32x32b.x16.pack::16b (32 columns -> 16 regs)
//         2: 32x32b.x32.pack::16b (64 columns -> 32 regs); 3: 16x256b.x4 (32 regs: 16 lanes x 64 cols... )
template <int MODE>
__global__ void __launch_bounds__(512, 1) ld_loop(int iters, unsigned long long* out) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) ptx::tmem_alloc<512>(&tslot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
  const int wq = warp >> 2;  // warps sharing a lane quarter split the columns
  uint32_t acc = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t col = (uint32_t)(((it + wq) * 64) & 511);
    uint32_t a[32], b[32];
    if (MODE == 0) {
      LD32("32x32b.x32", tmem + lane_base + col, a);
      LD32("32x32b.x32", tmem + lane_base + ((col + 32) & 511), b);
    } else if (MODE == 2) {
      LD32("32x32b.x32.pack::16b", tmem + lane_base + (col & ~63u), a);
      LD32("32x32b.x32.pack::16b", tmem + lane_base + ((col + 64) & 448u), b);
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) acc ^= a[i] + b[i];
  }
  const unsigned long long t1 = clock64();
  __syncthreads();
  if ((threadIdx.x & 31) == 0) atomicAdd(out, t1 - t0);
  if (acc == 0x12345678u) out[1] = acc;
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 0) ptx::tmem_dealloc<512>(tmem);
}

template <int MODE>
static void run(int warps, int iters) {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaMemset(d, 0, 16);
  ld_loop<MODE><<<148, warps * 32>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double cyc = (double)h[0] / (148.0 * warps);  // mean cycles per warp
  const int cols = MODE == 0 ? 64 : 128;              // columns per iteration per warp (2 loads)
  // TMEM cells (lanes x columns x 4 B) read per clock per SM
  const double bytes = (double)warps * iters * 32 * cols * 4;
  printf("{\"mode\": %d, \"warps\": %d, \"err\": \"%s\", \"cycles_per_warp\": %.0f, "
         "\"cell_bytes_per_clk_per_sm\": %.1f, \"reg_bytes_per_clk_per_sm\": %.1f}\n",
         MODE, warps, cudaGetErrorString(e), cyc, bytes / cyc, (MODE == 0 ? 1.0 : 0.5) * bytes / cyc);
  cudaFree(d);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<0>(w, 20000);
    run<2>(w, 20000);
  }
  return 0;
}
