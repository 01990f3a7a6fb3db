// Probe: tcgen05.cp.128x256b as an accumulator initialiser.  (1) layout: one
// 256-byte shared-memory block (two core matrices of 8 identical 16-byte rows)
// per 8 columns, SBO = 0 so all 16 row groups read the same block -> every TMEM
// lane gets the same 8 values; checked with tcgen05.ld.  (2) issue cost inside
// the screen kernel's per-tile MMA pattern (8 E4M3 K steps over two row tiles)
// with: the two augmented BF16 K steps (current kernel), 32 copies, nothing.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a scripts/tmem_cp_probe.cu -o build/tmem_cp_probe
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2501_05587_b200/csrc/tc_ptx.cuh"

using namespace pcb;

__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ __forceinline__ void umma_bf16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// the 4 KB source of one 128-column tile: block q (8 columns) at q * 256,
// core matrix h (columns 4h..4h+3) at + 128 h, 8 identical rows of 16 B
__device__ void fill_src(float* src, int tile) {
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
    const int q = i / 64, h = (i / 32) & 1, c = i & 3;
    src[i] = (float)(tile * 1000 + q * 8 + h * 4 + c) + 0.25f;
  }
}

template <int MODE>  // 0: layout check (LBO 128, SBO 0); 1: LBO 0 / SBO 128 (the other reading)
__global__ void cp_check(int* bad, float* sample) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  fill_src(reinterpret_cast<float*>(smem), 3);
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_barrier_init();
  }
  if (threadIdx.x < 32) ptx::tmem_alloc<512>(&tslot);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x < 32) {
    if (ptx::elect_one()) {
      for (int q = 0; q < 16; ++q) {
        const uint64_t d = MODE == 0 ? ptx::sdesc_k_none(ptx::smem_u32(smem + q * 256), 128, 0)
                                     : ptx::sdesc_k_none(ptx::smem_u32(smem + q * 256), 0, 128);
        tmem_cp_128x256b(tmem + 8 * q, d);
      }
      ptx::umma_commit(&bar);
    }
    __syncwarp();
  }
  ptx::mbar_wait(&bar, 0);
  ptx::tc_fence_after();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int nb = 0;
  for (int q = 0; q < 4; ++q) {
    uint32_t r[32];
    ptx::tmem_ld_32x32b_x32_async(tmem + ((uint32_t)(warp * 32) << 16) + 32 * q, r);
    ptx::tmem_wait_ld(r);
    for (int i = 0; i < 32; ++i) {
      const float want = 3000.0f + (float)(32 * q + i) + 0.25f;
      if (__uint_as_float(r[i]) != want) ++nb;
      if (warp * 32 + lane == 77) sample[32 * q + i] = __uint_as_float(r[i]);
    }
  }
  atomicAdd(bad, nb);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (threadIdx.x < 32) ptx::tmem_dealloc<512>(tmem);
}

// per tile: 8 E4M3 K=32 MMAs (two row tiles x 4 K steps, N = 128) plus
// INIT 0: 2 BF16 K=16 augmented MMAs; 1: 32 tcgen05.cp (16 per accumulator) before the MMAs; 2: nothing
template <int INIT>
__global__ void __launch_bounds__(128, 1) pattern(int iters, unsigned long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw & 1023u)) & 1023u);
  uint8_t* sA = smem;              // 2 row tiles x 16 KB
  uint8_t* sB = smem + 32768;      // 4 stages x 16 KB
  uint8_t* sX = smem + 98304;      // aug operands / copy source, 8 KB
  __shared__ uint64_t bar;
  __shared__ uint64_t bar2[2];
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 106496 / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u;
    h ^= h >> 15;
    h *= 0x85ebca6bu;
    h ^= h >> 13;
    reinterpret_cast<uint32_t*>(smem)[i] = h & 0x37373737u;  // small E4M3 / BF16 values
  }
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::mbar_init(&bar2[0], 1);
    ptx::mbar_init(&bar2[1], 1);
    ptx::fence_barrier_init();
  }
  if (threadIdx.x < 32) ptx::tmem_alloc<512>(&tslot);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x < 32) {
    const uint32_t idesc_8 = ptx::idesc_e4m3<128, 128>();
    const uint32_t idesc_h = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t a0 = ptx::sdesc_k_sw128(ptx::smem_u32(sA));
    const uint64_t a1 = ptx::sdesc_k_sw128(ptx::smem_u32(sA + 16384));
    const uint64_t bb = ptx::sdesc_k_sw128(ptx::smem_u32(sB));
    const uint64_t aa = ptx::sdesc_k_none(ptx::smem_u32(sX), 128 * 16, 128);
    const uint64_t ba = ptx::sdesc_k_none(ptx::smem_u32(sX + 4096), 128 * 16, 128);
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      ptx::tc_fence_after();
      if (ptx::elect_one()) {
        const uint32_t d = tmem + (it & 1) * 256;
        const uint64_t bs = bb + (uint64_t)(((it & 3) * 16384) >> 4);
        if (INIT == 1) {
          for (int q = 0; q < 16; ++q) {
            const uint64_t s = ptx::sdesc_k_none(ptx::smem_u32(sX + q * 256), 128, 0);
            tmem_cp_128x256b(d + 8 * q, s);
            tmem_cp_128x256b(d + 128 + 8 * q, s);
          }
        }
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint64_t off = (uint64_t)(ks * 32) >> 4;
          ptx::umma_f8(d, a0 + off, bs + off, idesc_8, INIT == 1 || ks != 0);
          ptx::umma_f8(d + 128, a1 + off, bs + off, idesc_8, INIT == 1 || ks != 0);
        }
        if (INIT == 0) {
          umma_bf16(d, aa, ba, idesc_h, 1u);
          umma_bf16(d + 128, aa, ba, idesc_h, 1u);
        }
        ptx::umma_commit(&bar2[0]);
        ptx::umma_commit(&bar2[1]);
      }
      __syncwarp();
    }
    if (ptx::elect_one()) ptx::umma_commit(&bar);
    __syncwarp();
    ptx::mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (threadIdx.x < 32) ptx::tmem_dealloc<512>(tmem);
}

template <int INIT>
static void run_pattern(int sms, int iters) {
  unsigned long long* cyc;
  cudaMalloc(&cyc, sms * sizeof(unsigned long long));
  const int smem = 106496 + 1024;
  cudaFuncSetAttribute(pattern<INIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  pattern<INIT><<<sms, 128, smem>>>(iters / 10, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  pattern<INIT><<<sms, 128, smem>>>(iters, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long c0;
  cudaMemcpy(&c0, cyc, sizeof(c0), cudaMemcpyDeviceToHost);
  printf("init=%s: %.3f ms, %.1f SM0 cycles per tile (2 row tiles)  err=%s\n",
         INIT == 0 ? "aug BF16 MMA x2" : INIT == 1 ? "tcgen05.cp x32" : "none", ms, (double)c0 / iters,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}

template <int MODE>
static void run_check() {
  int* bad;
  float* sample;
  cudaMalloc(&bad, 4);
  cudaMalloc(&sample, 128 * 4);
  cudaMemset(bad, 0, 4);
  cudaFuncSetAttribute(cp_check<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
  cp_check<MODE><<<1, 128, 8192>>>(bad, sample);
  int hb = -1;
  float hs[128];
  cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hs, sample, 512, cudaMemcpyDeviceToHost);
  printf("layout %s: %d of 16384 cells wrong  (lane 77 cols 0..11: %g %g %g %g %g %g %g %g %g %g %g %g) err=%s\n",
         MODE == 0 ? "LBO=128,SBO=0" : "LBO=0,SBO=128", hb, hs[0], hs[1], hs[2], hs[3], hs[4], hs[5], hs[6], hs[7],
         hs[8], hs[9], hs[10], hs[11], cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run_check<0>();
  run_check<1>();
  for (int r = 0; r < 2; ++r) {
    run_pattern<0>(sms, 100000);
    run_pattern<1>(sms, 100000);
    run_pattern<2>(sms, 100000);
  }
  return 0;
}
