// Microbenchmark: issue rate of tcgen05.mma kind::tf32 vs kind::f16 (bf16) on
// one B200, operands resident in shared memory, accumulators in TMEM.  One CTA
// per SM, one elected thread issues back-to-back MMAs (M=128, N=256).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a scripts/mma_peak.cu -o build/mma_peak
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2501_05587_b200/csrc/tc_ptx.cuh"

using namespace pcb;

constexpr int M = 128, N = 256;

__device__ __forceinline__ void umma_bf16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

template <bool TF32>
__global__ void __launch_bounds__(128, 1) mma_loop(int iters, unsigned long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw & 1023u)) & 1023u);
  uint8_t* sA = smem;                 // 128 rows x 128 B
  uint8_t* sB = smem + 16384;         // 256 rows x 128 B
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.0f;
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
    const uint64_t a = ptx::sdesc_k_sw128(ptx::smem_u32(sA));
    const uint64_t b = ptx::sdesc_k_sw128(ptx::smem_u32(sB));
    const uint32_t idesc_t = ptx::idesc_tf32<M, N>();
    const uint32_t idesc_h = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    unsigned long long t0 = clock64();
    if (ptx::elect_one()) {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint64_t off = (uint64_t)(ks * 32) >> 4;
          if (TF32) ptx::umma_tf32(tmem, a + off, b + off, idesc_t, (it | ks) != 0);
          else umma_bf16(tmem, a + off, b + off, idesc_h, (it | ks) != 0);
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

template <bool TF32>
static void run(int sms, int iters) {
  unsigned long long* cyc;
  cudaMalloc(&cyc, sms * sizeof(unsigned long long));
  const int smem = 16384 + 32768 + 1024;
  cudaFuncSetAttribute(mma_loop<TF32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_loop<TF32><<<sms, 128, smem>>>(iters / 10, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mma_loop<TF32><<<sms, 128, smem>>>(iters, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long c0;
  cudaMemcpy(&c0, cyc, sizeof(c0), cudaMemcpyDeviceToHost);
  // K per instruction: tf32 8, bf16 16; 4 instructions per iteration
  const double k_per = TF32 ? 8.0 : 16.0;
  const double flops = (double)sms * iters * 4 * 2.0 * M * N * k_per;
  printf("%s: %.3f ms, %.1f TFLOP/s, %.1f flop/cycle/SM (SM0 cycles %llu)  err=%s\n", TF32 ? "kind::tf32" : "kind::f16 (bf16)",
         ms, flops / (ms * 1e-3) / 1e12, (double)iters * 4 * 2.0 * M * N * k_per / (double)c0, c0,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int r = 0; r < 2; ++r) {
    run<true>(sms, 200000);
    run<false>(sms, 200000);
  }
  return 0;
}
