// Shared pieces of the certified-screening kernels (assign_screen*.cu).
#pragma once
#include <cudaTypedefs.h>

#include "pcb_common.cuh"
#include "tc_ptx.cuh"

namespace pcb {

constexpr int SC_BK = 32;       // f32 per 128-byte swizzle row (one K chunk)
constexpr int SC_KMAX = 6144;   // smem copy of the shifted centroid norms (k <= 6144)

// chunk-local column ids; held in registers so (key & ~31) | id is a single LOP3
static __constant__ uint32_t kChunkIds[32] = {0,  1,  2,  3,  4,  5,  6,  7,  8,  9,  10, 11, 12, 13, 14, 15,
                                       16, 17, 18, 19, 20, 21, 22, 23, 24, 25, 26, 27, 28, 29, 30, 31};

__device__ __forceinline__ float fmin3(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

__device__ __forceinline__ float pack_idx(float key, uint32_t i) {
  return __uint_as_float((__float_as_uint(key) & 0xFFFFFFE0u) | i);
}


// Rigorous per-row bound 2E on |key_j - OFF - s_j| (assign_screen.cu header).
__device__ __forceinline__ float screen_two_e(float an, float dan, float Bmax, float dBmax, float OFF,
                                              float acc_rel) {
  const float gerr = dan * Bmax + an * dBmax + dan * dBmax + acc_rel * an * Bmax;
  const float cbn = Bmax + dBmax;
  const float kmax = OFF + 2.0f * (an + dan) * cbn + cbn * cbn;
  return 2.0f * 1.0001f * (2.0f * gerr + 0x1p-16f * kmax);
}

// One 32-column chunk of accumulators v[] (overwritten with the keys): update
// the running packed min R1 (index r1) and the count of keys within twoE of it.
__device__ __forceinline__ void screen_chunk(float (&v)[32], const float* __restrict__ cprime_chunk,
                                             const uint32_t (&cid)[32], int col0, float twoE, float big,
                                             float& R1, int& r1, float& cnt) {
  const float4* cp4 = reinterpret_cast<const float4*>(cprime_chunk);
  float ma = 3.4e38f, mb = 3.4e38f;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float4 c4 = cp4[q];
    v[4 * q + 0] = fmaf(-2.0f, v[4 * q + 0], c4.x);
    v[4 * q + 1] = fmaf(-2.0f, v[4 * q + 1], c4.y);
    v[4 * q + 2] = fmaf(-2.0f, v[4 * q + 2], c4.z);
    v[4 * q + 3] = fmaf(-2.0f, v[4 * q + 3], c4.w);
    const float k0 = __uint_as_float((__float_as_uint(v[4 * q + 0]) & 0xFFFFFFE0u) | cid[4 * q + 0]);
    const float k1 = __uint_as_float((__float_as_uint(v[4 * q + 1]) & 0xFFFFFFE0u) | cid[4 * q + 1]);
    const float k2 = __uint_as_float((__float_as_uint(v[4 * q + 2]) & 0xFFFFFFE0u) | cid[4 * q + 2]);
    const float k3 = __uint_as_float((__float_as_uint(v[4 * q + 3]) & 0xFFFFFFE0u) | cid[4 * q + 3]);
    ma = fmin3(ma, k0, k1);
    mb = fmin3(mb, k2, k3);
  }
  const float m = fminf(ma, mb);
  // (a) much better min: every earlier counted key is above the new threshold;
  // (b) slightly better: the old min stays within it, so the row is ambiguous
  //     whatever the over-count
  if (m < R1 - twoE) cnt = 0.0f;
  if (m < R1) {
    R1 = m;
    r1 = col0 + (int)(__float_as_uint(m) & 31u);
  }
  const float thr = R1 + twoE + 0x1p-16f * fabsf(R1);
  const float thr_big = thr * big;
  float c0 = 0.0f, c1 = 0.0f;
#pragma unroll
  for (int i = 0; i < 32; i += 2) {
    c0 += __saturatef(fmaf(v[i], -big, thr_big));
    c1 += __saturatef(fmaf(v[i + 1], -big, thr_big));
  }
  cnt += c0 + c1;
}

// Append ambiguous rows to the list (warp-aggregated atomic).
__device__ __forceinline__ void screen_append(bool amb, int64_t row, int* amb_list, int* amb_count, int lane) {
  const unsigned msk = __ballot_sync(0xffffffffu, amb);
  if (msk) {
    int base = 0;
    if (lane == 0) base = atomicAdd(amb_count, __popc(msk));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (amb) amb_list[base + __popc(msk & ((1u << lane) - 1u))] = (int)row;
  }
}

static inline int make_tmap_rows(CUtensorMap* m, const float* base, int64_t rows, int cols, int box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (enc == nullptr) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return PCB_ENODEV;
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * sizeof(float)};
  cuuint32_t box[2] = {(cuuint32_t)SC_BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : PCB_EINVAL;
}


}  // namespace pcb
