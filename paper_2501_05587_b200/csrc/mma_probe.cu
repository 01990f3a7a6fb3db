// Accumulation probe of the tensor core (test infrastructure for the
// certificates of the screening kernels, not on the Lloyd path).
//
// The certified screens (assign_screen_bf16.cu, assign_screen.cu) bound the
// error of the f32 accumulation inside tcgen05.mma by an assumed model: each
// MMA of K products adds at most a fixed multiple of 2^-23 of the sum of the
// |terms| it combines (the running accumulator included).  Nothing in the PTX
// documentation states how kind::f8f6f4 / kind::f16 / kind::tf32 actually
// align, truncate or round inside one MMA, so this kernel runs one chain of
// MMAs (M = N = 128, 32 bytes of K per step, F32 accumulator in TMEM,
// optionally preloaded with an arbitrary f32 matrix) on caller-chosen
// operands and returns the accumulator; tests/test_gpu_mma_probe.py compares
// it with the exactly rounded sums and checks the screens' budget.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "pcb_common.cuh"
#include "pcb_launch.cuh"
#include "tc_ptx.cuh"

namespace pcb {

constexpr int MP_BATCH = 16;              // K steps staged in shared memory at a time
constexpr uint32_t MP_STEP = 128 * 32;    // one operand's bytes per step (128 rows x 32 B)
constexpr uint32_t MP_SMEM = 1024 + 2 * MP_BATCH * MP_STEP;

// A, B: 128 rows of nsteps * 32 bytes (row-major, K contiguous).  Step s
// multiplies bytes [32 s, 32 s + 32) of every row with kind kinds[s]:
// 0 = E4M3 x E4M3 (kind::f8f6f4, K = 32), 1 = BF16 x BF16 (kind::f16, K = 16),
// 2 = TF32 x TF32 (kind::tf32, K = 8).  D (128 x 128 f32) = init + sum of the
// steps, or the sum alone when init is null.
// H16: every step is E4M3 (kind::f8f6f4) into an F16 accumulator; init and D
// go through tcgen05.st/ld .unpack/.pack::16b (two 16-bit columns per
// register), raw (optional) receives the unpacked 32-bit TMEM cells.
template <bool H16>
__global__ void __launch_bounds__(128, 1)
mma_probe_kernel(const uint8_t* __restrict__ A, const uint8_t* __restrict__ B, const int* __restrict__ kinds,
                 int nsteps, const float* __restrict__ init, float* __restrict__ D, uint32_t* __restrict__ raw_out) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t raw = ptx::smem_u32(smem_raw);
  uint8_t* sA = smem_raw + ((1024u - (raw & 1023u)) & 1023u);
  uint8_t* sB = sA + MP_BATCH * MP_STEP;
  const int warp = threadIdx.x >> 5, row = threadIdx.x;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 0) ptx::tmem_alloc<128>(&tslot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  if (init != nullptr) {
    if (H16) {
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        uint32_t r[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const __half2 h = __floats2half2_rn(init[row * 128 + c * 64 + 2 * i], init[row * 128 + c * 64 + 2 * i + 1]);
          r[i] = *reinterpret_cast<const uint32_t*>(&h);
        }
        ptx::tmem_st_32x32b_x32_unpack16(trow + 64 * c, r);
      }
    } else {
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(init[row * 128 + c * 32 + i]);
        ptx::tmem_st_32x32b_x32(trow + 32 * c, r);
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const int64_t ld = (int64_t)nsteps * 32;
  uint32_t phase = 0;
  for (int s0 = 0; s0 < nsteps; s0 += MP_BATCH) {
    const int nb = nsteps - s0 < MP_BATCH ? nsteps - s0 : MP_BATCH;
    // no-swizzle K-major core layout per step: [2 K halves][128 rows][16 B]
    for (int s = 0; s < nb; ++s) {
      const uint4* ga = reinterpret_cast<const uint4*>(A + row * ld + (int64_t)(s0 + s) * 32);
      const uint4* gb = reinterpret_cast<const uint4*>(B + row * ld + (int64_t)(s0 + s) * 32);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        *reinterpret_cast<uint4*>(sA + s * MP_STEP + h * 2048 + row * 16) = ga[h];
        *reinterpret_cast<uint4*>(sB + s * MP_STEP + h * 2048 + row * 16) = gb[h];
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 0) {
      if (ptx::elect_one()) {
        for (int s = 0; s < nb; ++s) {
          const uint64_t ad = ptx::sdesc_k_none(ptx::smem_u32(sA + s * MP_STEP), 2048, 128);
          const uint64_t bd = ptx::sdesc_k_none(ptx::smem_u32(sB + s * MP_STEP), 2048, 128);
          const uint32_t acc = (init != nullptr || s0 + s > 0) ? 1u : 0u;
          const int kind = kinds[s0 + s];
          if (H16) ptx::umma_f8(tmem, ad, bd, ptx::idesc_e4m3<128, 128>() & ~(3u << 4), acc);  // D format F16
          else if (kind == 0) ptx::umma_f8(tmem, ad, bd, ptx::idesc_e4m3<128, 128>(), acc);
          else if (kind == 1) ptx::umma_f16(tmem, ad, bd, ptx::idesc_bf16<128, 128>(), acc);
          else ptx::umma_tf32(tmem, ad, bd, ptx::idesc_tf32<128, 128>(), acc);
        }
        ptx::umma_commit(&bar);
      }
      __syncwarp();
    }
    ptx::mbar_wait(&bar, phase);
    phase ^= 1u;
    ptx::tc_fence_after();
    __syncthreads();  // the next batch overwrites the operands the MMAs read
  }
  if (H16) {
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      uint32_t r[32];
      ptx::tmem_ld_32x32b_x32_async_pack16(trow + 64 * c, r);
      ptx::tmem_wait_ld(r);
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&r[i]));
        D[row * 128 + c * 64 + 2 * i] = f.x;
        D[row * 128 + c * 64 + 2 * i + 1] = f.y;
      }
    }
    if (raw_out != nullptr) {
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        float v[32];
        ptx::tmem_ld_32x32b_x32(trow + 32 * c, v);
#pragma unroll
        for (int i = 0; i < 32; ++i) raw_out[row * 128 + c * 32 + i] = __float_as_uint(v[i]);
      }
    }
  } else {
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      float v[32];
      ptx::tmem_ld_32x32b_x32(trow + 32 * c, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) D[row * 128 + c * 32 + i] = v[i];
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 0) ptx::tmem_dealloc<128>(tmem);
}

}  // namespace pcb

using namespace pcb;

extern "C" int pcb_mma_probe(const void* A, const void* B, const int* kinds, int nsteps, const float* init,
                             float* D, void* stream) {
  if (!A || !B || !kinds || !D || nsteps < 1 || nsteps > 4096) return PCB_EINVAL;
  cudaError_t e = cudaFuncSetAttribute(mma_probe_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)MP_SMEM);
  if (e != cudaSuccess) return (int)e;
  mma_probe_kernel<false><<<1, 128, MP_SMEM, (cudaStream_t)stream>>>((const uint8_t*)A, (const uint8_t*)B, kinds,
                                                                     nsteps, init, D, nullptr);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_mma_probe_f16acc(const void* A, const void* B, const int* kinds, int nsteps, const float* init,
                                    float* D, uint32_t* raw, void* stream) {
  if (!A || !B || !kinds || !D || nsteps < 1 || nsteps > 4096) return PCB_EINVAL;
  cudaError_t e = cudaFuncSetAttribute(mma_probe_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)MP_SMEM);
  if (e != cudaSuccess) return (int)e;
  mma_probe_kernel<true><<<1, 128, MP_SMEM, (cudaStream_t)stream>>>((const uint8_t*)A, (const uint8_t*)B, kinds,
                                                                    nsteps, init, D, raw);
  PCB_CHECK_LAUNCH();
  return 0;
}
