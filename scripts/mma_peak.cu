// Microbenchmark: issue rate of tcgen05.mma kind::tf32 / kind::f16 (bf16) /
// kind::f8f6f4 (e4m3) on one B200, operands resident in shared memory (SS
// mode), accumulators in TMEM.  One CTA per SM, one elected thread issues
// back-to-back MMAs (M=128, N=128 or 256).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a scripts/mma_peak.cu -o build/mma_peak
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2501_05587_b200/csrc/tc_ptx.cuh"

using namespace pcb;

constexpr int M = 128;

__device__ __forceinline__ void umma_bf16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// KIND: 0 tf32, 1 bf16, 2 e4m3
// KIND 3: the screen kernel's issue pattern per centroid tile — 4 E4M3 K steps
// alternating between two row tiles / accumulators, then one BF16 K=16 step
// per row tile (the augmented step)
template <int KIND, int N, bool RAND>
__global__ void __launch_bounds__(128, 1) mma_loop(int iters, unsigned long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw & 1023u)) & 1023u);
  uint8_t* sA = smem;                 // 128 rows x 128 B
  uint8_t* sB = smem + 16384;         // 256 rows x 128 B
  __shared__ uint64_t bar;
  __shared__ uint64_t bar2[2];
  __shared__ uint32_t tslot;
  // RAND: pseudo-random operand bytes (E4M3 / BF16 values of both signs) instead of zeros
  for (int i = threadIdx.x; i < (16384 * 8) / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u;
    h ^= h >> 15;
    h *= 0x85ebca6bu;
    h ^= h >> 13;
    // RAND: E4M3 bytes of every sign / exponent / mantissa except the NaN codes (bit 3 cleared)
    reinterpret_cast<uint32_t*>(smem)[i] = RAND ? (h & 0xf7f7f7f7u) : 0u;
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
    const uint64_t a = ptx::sdesc_k_sw128(ptx::smem_u32(sA));
    const uint64_t b = ptx::sdesc_k_sw128(ptx::smem_u32(sB));
    const uint32_t idesc_t = ptx::idesc_tf32<M, N>();
    const uint32_t idesc_h = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint32_t idesc_8 = ptx::idesc_e4m3<M, N>();
    const uint64_t a5 = ptx::sdesc_k_sw128(ptx::smem_u32(sA + 32768 + 65536));  // second A tile
    const uint64_t b5 = ptx::sdesc_k_sw128(ptx::smem_u32(sA + 32768));          // 4 B stages of 16 KB
    unsigned long long t0 = clock64();
    if (KIND >= 6) {
      // KIND 6: the kernel's issue structure — whole warp loops, fence after
      // thread sync, one elected lane issues the tile's 10 MMAs + 2 commits
      for (int it = 0; it < iters; ++it) {
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint64_t off = (uint64_t)(ks * 32) >> 4;
            const uint64_t bs = b5 + (uint64_t)(((it & 3) * 16384) >> 4) + off;
            ptx::umma_f8(tmem + (it & 1) * 256, a + off, bs, idesc_8, ks != 0);
            ptx::umma_f8(tmem + (it & 1) * 256 + 128, a5 + off, bs, idesc_8, ks != 0);
          }
          const uint64_t aa = ptx::sdesc_k_none(ptx::smem_u32(sA), 128 * 16, 128);
          const uint64_t ba = ptx::sdesc_k_none(ptx::smem_u32(sB), N * 16, 128);
          umma_bf16(tmem + (it & 1) * 256, aa, ba, idesc_h, 1u);
          umma_bf16(tmem + (it & 1) * 256 + 128, aa, ba, idesc_h, 1u);
          ptx::umma_commit(&bar2[0]);
          ptx::umma_commit(&bar2[1]);
        }
        __syncwarp();
      }
      if (ptx::elect_one()) ptx::umma_commit(&bar);
      __syncwarp();
    } else if (ptx::elect_one()) {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint64_t off = (uint64_t)(ks * 32) >> 4;
          if (KIND == 0) ptx::umma_tf32(tmem, a + off, b + off, idesc_t, (it | ks) != 0);
          else if (KIND == 1) umma_bf16(tmem, a + off, b + off, idesc_h, (it | ks) != 0);
          else if (KIND == 2) ptx::umma_f8(tmem, a + off, b + off, idesc_8, (it | ks) != 0);
          else if (KIND < 5) {  // KIND 3 / 4
            ptx::umma_f8(tmem + (it & 1) * 256, a + off, b + off, idesc_8, ks != 0);
            ptx::umma_f8(tmem + (it & 1) * 256 + 128, a + off, b + off, idesc_8, ks != 0);
          } else {  // KIND 5: distinct operands — two A row tiles, B rotating over 4 stages
            ptx::umma_f8(tmem + (it & 1) * 256, a + off, b5 + (uint64_t)(((it & 3) * 16384) >> 4) + off, idesc_8, ks != 0);
            ptx::umma_f8(tmem + (it & 1) * 256 + 128, a5 + off, b5 + (uint64_t)(((it & 3) * 16384) >> 4) + off, idesc_8, ks != 0);
          }
        }
        if (KIND >= 3) {
          const uint64_t aa = ptx::sdesc_k_none(ptx::smem_u32(sA), 128 * 16, 128);
          const uint64_t ba = ptx::sdesc_k_none(ptx::smem_u32(sB), N * 16, 128);
          umma_bf16(tmem + (it & 1) * 256, aa, ba, idesc_h, 1u);
          umma_bf16(tmem + (it & 1) * 256 + 128, aa, ba, idesc_h, 1u);
          // KIND 4: + the kernel's per-tile commits (stage release + accumulator ready)
          if (KIND == 4) { ptx::umma_commit(&bar2[0]); ptx::umma_commit(&bar2[1]); }
        }
      }
      ptx::umma_commit(&bar);
    }
    __syncwarp();
    ptx::mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (threadIdx.x < 32) ptx::tmem_dealloc<512>(tmem);
}

template <int KIND, int N, bool RAND = false>
static void run(int sms, int iters) {
  unsigned long long* cyc;
  cudaMalloc(&cyc, sms * sizeof(unsigned long long));
  const int smem = 16384 * 8 + 1024;
  cudaFuncSetAttribute(mma_loop<KIND, N, RAND>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_loop<KIND, N, RAND><<<sms, 128, smem>>>(iters / 10, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mma_loop<KIND, N, RAND><<<sms, 128, smem>>>(iters, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long c0;
  cudaMemcpy(&c0, cyc, sizeof(c0), cudaMemcpyDeviceToHost);
  // K per instruction: tf32 8, bf16 16; 4 instructions per iteration
  const double k_per = KIND == 0 ? 8.0 : KIND == 1 ? 16.0 : 32.0;
  // KIND 3 counts the E4M3 work only (2 row tiles x 4 steps; the BF16 step is overhead)
  const double flops = (double)sms * iters * (KIND >= 3 ? 8 : 4) * 2.0 * M * N * k_per;
  printf("%s N=%d: %.3f ms, %.1f TFLOP/s, %.1f flop/cycle/SM (SM0 cycles %llu)  err=%s\n", KIND == 0 ? "kind::tf32" : KIND == 1 ? "kind::f16 (bf16)" : KIND == 2 ? "kind::f8f6f4 (e4m3)" : (KIND == 6 ? "kernel issue structure (warp loop, fence, elect, commits)" : KIND == 5 ? "screen pattern, distinct A/B tiles, random data" : KIND == 4 ? "screen pattern + 2 commits per tile, random data" : RAND ? "screen pattern e4m3+bf16 aug, random data" : "screen pattern e4m3+bf16 aug"),
         N, ms, flops / (ms * 1e-3) / 1e12, (double)iters * (KIND >= 3 ? 8 : 4) * 2.0 * M * N * k_per / (double)c0, c0,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int r = 0; r < 1; ++r) {
    run<0, 256>(sms, 200000);
    run<1, 256>(sms, 200000);
    run<2, 256>(sms, 200000);
    run<1, 128>(sms, 200000);
    run<2, 128>(sms, 200000);
    run<2, 128, true>(sms, 200000);
    run<1, 128, true>(sms, 200000);
    run<3, 128>(sms, 100000);
    run<3, 128, true>(sms, 100000);
    run<4, 128, true>(sms, 100000);
    run<5, 128, true>(sms, 100000);
    run<5, 128, false>(sms, 100000);
    run<6, 128, true>(sms, 100000);
  }
  return 0;
}
