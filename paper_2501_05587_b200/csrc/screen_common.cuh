// Shared pieces of the certified-screening kernels (assign_screen*.cu).
#pragma once
#include <cudaTypedefs.h>

#include "pcb_common.cuh"
#include "tc_ptx.cuh"

namespace pcb {

constexpr int SC_BK = 32;       // f32 per 128-byte swizzle row (one K chunk)
constexpr int SC_KMAX = 6144;   // smem copy of the shifted centroid norms (k <= 6144)

// ~31 read from constant memory so the compiler cannot fold (key & ~31) | id
// into two immediates: with the mask in a register the pack is one LOP3
static __constant__ uint32_t kIdxMask = 0xFFFFFFE0u;

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

// Same bound when the MMA itself adds |c|^2 + OFF (augmented K step): the
// f32 accumulation error also scales with the key magnitude (acc_rel * kmax).
__device__ __forceinline__ float screen_two_e_aug(float an, float dan, float Bmax, float dBmax, float OFF,
                                                  float acc_rel) {
  const float gerr = dan * Bmax + an * dBmax + dan * dBmax + acc_rel * an * Bmax;
  const float cbn = Bmax + dBmax;
  const float kmax = OFF + 2.0f * (an + dan) * cbn + cbn * cbn;
  return 2.0f * 1.0001f * (2.0f * gerr + (0x1p-16f + acc_rel) * kmax);
}

// Packed f32x2 helpers (FFMA2 / FADD2 on sm_100a: two lanes per issue slot).
__device__ __forceinline__ unsigned long long f2pack(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2unpack(unsigned long long r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ unsigned long long fadd2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// Shifted centroid norms c'_j of one 32-column chunk, smem -> registers.
__device__ __forceinline__ void load_cprime(float (&cp)[32], const float* __restrict__ cprime_chunk) {
  const float4* cp4 = reinterpret_cast<const float4*>(cprime_chunk);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
#if defined(PCB_EXP) && PCB_EXP == 3
    const float4 c4 = make_float4(1.0f * q, 2.0f * q, 3.0f + q, 4.0f + q);  // experiment: no smem reads
#else
    const float4 c4 = cp4[q];
#endif
    cp[4 * q + 0] = c4.x;
    cp[4 * q + 1] = c4.y;
    cp[4 * q + 2] = c4.z;
    cp[4 * q + 3] = c4.w;
  }
}

// One 32-column chunk of accumulators v[] (overwritten with the keys) and its
// shifted centroid norms cp[]: update the running packed min R1 (index r1) and
// the count of keys within twoE of it.
// Per element: 1/2 FFMA2 (key), 1 LOP3 (index pack), 1/2 FMNMX3, 1 FFMA.SAT and
// 1/2 FADD2 (count) — the epilogue is issue-bound, so the f32x2 forms matter.
// `msk` is ~31 held in a register so the pack is one LOP3 with the id immediate.
__device__ __forceinline__ void screen_update(const float (&v)[32], float m, int col0, float twoE, float big,
                                              float& R1, int& r1, float& cnt);

// Full update of one chunk of keys v[] with the running best two packed keys
// (R1, r1), (R2, r2) and an exact integer count of keys within the threshold
// (so that cnt == 2 identifies rows whose candidates are exactly r1 and r2:
// an over-count only happens when the minimum dropped by less than 2E, and
// then the old minimum is itself within the final threshold).
__device__ __forceinline__ void screen_chunk_top2(const float (&v)[32], uint32_t msk, int col0, float twoE, float& R1,
                                                  int& r1, float& R2, int& r2, float& cnt) {
  float ma = 3.4e38f, mb = 3.4e38f;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float k0 = __uint_as_float((__float_as_uint(v[4 * q + 0]) & msk) | (uint32_t)(4 * q + 0));
    const float k1 = __uint_as_float((__float_as_uint(v[4 * q + 1]) & msk) | (uint32_t)(4 * q + 1));
    const float k2 = __uint_as_float((__float_as_uint(v[4 * q + 2]) & msk) | (uint32_t)(4 * q + 2));
    const float k3 = __uint_as_float((__float_as_uint(v[4 * q + 3]) & msk) | (uint32_t)(4 * q + 3));
    ma = fmin3(ma, k0, k1);
    mb = fmin3(mb, k2, k3);
  }
  const float m = fminf(ma, mb);
  // second smallest packed key of the chunk (packed keys are distinct)
  float sa = 3.4e38f, sb = 3.4e38f;
#pragma unroll
  for (int i = 0; i < 32; i += 2) {
    const float k0 = __uint_as_float((__float_as_uint(v[i]) & msk) | (uint32_t)i);
    const float k1 = __uint_as_float((__float_as_uint(v[i + 1]) & msk) | (uint32_t)(i + 1));
    sa = fminf(sa, k0 == m ? 3.4e38f : k0);
    sb = fminf(sb, k1 == m ? 3.4e38f : k1);
  }
  const float m2 = fminf(sa, sb);
  if (m < R1 - twoE) cnt = 0.0f;
  if (m < R1) {
    if (m2 < R1) { R2 = m2; r2 = col0 + (int)(__float_as_uint(m2) & 31u); }
    else { R2 = R1; r2 = r1; }
    R1 = m;
    r1 = col0 + (int)(__float_as_uint(m) & 31u);
  } else if (m < R2) {
    R2 = m;
    r2 = col0 + (int)(__float_as_uint(m) & 31u);
  }
  const float thr = R1 + twoE + 0x1p-16f * fabsf(R1);
  float c = 0.0f;
#pragma unroll
  for (int i = 0; i < 32; ++i) c += v[i] <= thr ? 1.0f : 0.0f;
  cnt += c;
}

// Same on keys already formed (v[i] = cp[i] - 2 acc[i]).
__device__ __forceinline__ void screen_chunk_keys(const float (&v)[32], uint32_t msk, int col0, float twoE, float big,
                                                  float& R1, int& r1, float& cnt) {
  float ma = 3.4e38f, mb = 3.4e38f;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float k0 = __uint_as_float((__float_as_uint(v[4 * q + 0]) & msk) | (uint32_t)(4 * q + 0));
    const float k1 = __uint_as_float((__float_as_uint(v[4 * q + 1]) & msk) | (uint32_t)(4 * q + 1));
    const float k2 = __uint_as_float((__float_as_uint(v[4 * q + 2]) & msk) | (uint32_t)(4 * q + 2));
    const float k3 = __uint_as_float((__float_as_uint(v[4 * q + 3]) & msk) | (uint32_t)(4 * q + 3));
    ma = fmin3(ma, k0, k1);
    mb = fmin3(mb, k2, k3);
  }
  screen_update(v, fminf(ma, mb), col0, twoE, big, R1, r1, cnt);
}

// Running-min / ambiguity-count update of one chunk with packed minimum m.
__device__ __forceinline__ void screen_update(const float (&v)[32], float m, int col0, float twoE, float big,
                                              float& R1, int& r1, float& cnt) {
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
  unsigned long long c2 = 0ull, d2 = 0ull;
#pragma unroll
  for (int i = 0; i < 32; i += 4) {
    c2 = fadd2(c2, f2pack(__saturatef(fmaf(v[i], -big, thr_big)), __saturatef(fmaf(v[i + 1], -big, thr_big))));
    d2 = fadd2(d2, f2pack(__saturatef(fmaf(v[i + 2], -big, thr_big)), __saturatef(fmaf(v[i + 3], -big, thr_big))));
  }
  float x0, x1;
  f2unpack(fadd2(c2, d2), x0, x1);
  cnt += x0 + x1;
}

__device__ __forceinline__ void screen_chunk_regs(float (&v)[32], const float (&cp)[32], uint32_t msk, int col0,
                                                  float twoE, float big, float& R1, int& r1, float& cnt) {
  const unsigned long long m2 = f2pack(-2.0f, -2.0f);
  float ma = 3.4e38f, mb = 3.4e38f;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const unsigned long long a = ffma2(f2pack(v[4 * q + 0], v[4 * q + 1]), m2, f2pack(cp[4 * q + 0], cp[4 * q + 1]));
    const unsigned long long b = ffma2(f2pack(v[4 * q + 2], v[4 * q + 3]), m2, f2pack(cp[4 * q + 2], cp[4 * q + 3]));
    f2unpack(a, v[4 * q + 0], v[4 * q + 1]);
    f2unpack(b, v[4 * q + 2], v[4 * q + 3]);
    const float k0 = __uint_as_float((__float_as_uint(v[4 * q + 0]) & msk) | (uint32_t)(4 * q + 0));
    const float k1 = __uint_as_float((__float_as_uint(v[4 * q + 1]) & msk) | (uint32_t)(4 * q + 1));
    const float k2 = __uint_as_float((__float_as_uint(v[4 * q + 2]) & msk) | (uint32_t)(4 * q + 2));
    const float k3 = __uint_as_float((__float_as_uint(v[4 * q + 3]) & msk) | (uint32_t)(4 * q + 3));
    ma = fmin3(ma, k0, k1);
    mb = fmin3(mb, k2, k3);
  }
  screen_update(v, fminf(ma, mb), col0, twoE, big, R1, r1, cnt);
}

__device__ __forceinline__ void screen_chunk(float (&v)[32], const float* __restrict__ cprime_chunk, uint32_t msk,
                                             int col0, float twoE, float big, float& R1, int& r1, float& cnt) {
  float cp[32];
  load_cprime(cp, cprime_chunk);
  screen_chunk_regs(v, cp, msk, col0, twoE, big, R1, r1, cnt);
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
