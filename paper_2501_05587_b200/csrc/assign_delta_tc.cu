// delta-chunked P.C.P^T distance stage on the tcgen05 tensor cores — the
// tensor-core form of the ablation in PAPER.md:146-237 (the SIMT form is
// assign_delta.cu).
//
// The attachment writes the squared distance of point p to centroid c as the
// bilinear form q C q^T with q = [1, p] and the augmented (d+1) x (d+1)
// C = [[|c|^2, -c^T], [-c, I]] (analysis.py:83-102), pads r = d+1 to a
// multiple of delta, cuts C and P into delta x delta blocks, forms
// D_i = P_i C P_i^T block by block and keeps only the diagonal.  Its
// observation is that C_ab = 0 for a, b > 1, a != b, so per
// block column b only three block products survive (0-based block indices):
//
//   T_0 = sum_a Q_a C_a0                 (first block column, every a)
//   T_b = Q_0 C_0b + Q_b C_bb   (b > 0)  (first block row + diagonal block)
//   D   = sum_b rowdot(T_b, Q_b)         (diag of the block product)
//
// and the attachment's cost claim is that with tensor cores a
// block product P_ab C_ij costs O(1), i.e. a delta^2 gain over the scalar form.
// This kernel issues exactly those block products as tcgen05 MMAs, delta = 8
// (kind::tf32, K = 8), batched over 16 centroids along N (N = 16 * delta =
// 128: the B operand of one MMA is the column of 16 centroids' delta x delta
// blocks), M = 128 points:
//
//   Q_b . F_b -> T_0   F_b row (j, v), col u = C_j[8b+u][v]   (C_b0 blocks)
//   Q_0 . G_b -> T_b   G_b row (j, v), col u = C_j[u][8b+v]   (C_0b blocks)
//   Q_b . H   -> T_b   H   row (j, v), col u = [u == v]       (C_bb = I, b > 0)
//
// each product in 3xTF32 (hi.hi + hi.lo + lo.hi; the identity is exact in
// TF32, so Q_b . H needs only hi.I + lo.I), so labels stay FP32-faithful.
// The diagonal extraction rowdot(T_b, Q_b) is not a GEMM: the epilogue reads
// every T_b (128 rows x 128 columns of TMEM) and does delta FMAs per
// (point, centroid) with the point's q_b read from the staged A tile.
//
// Structure (one CTA per SM, persistent over 128-point tiles; 16-centroid
// groups inner):
//   warp 0     TMA: per (tile, group, 32-column chunk = 4 blocks) Q_hi, Q_lo,
//              F_hi, F_lo, G_hi, G_lo (128 rows x 128 B each, SWIZZLE_128B)
//              into a 2-stage ring; Q_0 (hi, lo) once per tile (no swizzle).
//   warp 1     MMA issuer: T_0 (2 TMEM buffers) and T_b (2 TMEM buffers).
//   warp 2     TMEM allocator; warp 3 builds H.
//   warps 4-7  epilogue: thread = point; D_j += rowdot(T_b, q_b) for the 16
//              centroids of the group, then the running (min, lowest j) and the
//              bookkeeping of _assignment_step (clustering.py:142-150).
// A stage is released by the MMA commit and by the 4 epilogue warps (they
// read q_b from it).
#include <cudaTypedefs.h>

#include "pcb_common.cuh"
#include "pcb_launch.cuh"
#include "tc_ptx.cuh"

namespace pcb {

namespace dtc {
constexpr int kDelta = 8;                  // block size delta (= TF32 MMA K)
constexpr int kBM = 128;                   // points per tile (UMMA M)
constexpr int kNc = 16;                    // centroids per group
constexpr int kBN = kNc * kDelta;          // UMMA N = 128
constexpr int kChunk = 32;                 // f32 columns per 128-byte swizzle row = 4 blocks
constexpr int kStages = 2;
constexpr int kThreads = 256;
constexpr int kHistMax = 4096;
constexpr uint32_t kTile = kBM * kChunk * 4;           // 16 KB (A and B tiles alike: 128 rows)
constexpr uint32_t kStageBytes = 6 * kTile;            // Q hi/lo, F hi/lo, G hi/lo
constexpr uint32_t kA0Bytes = 2 * kBM * kDelta * 4;    // Q_0 hi + lo, no swizzle
constexpr uint32_t kHBytes = kBN * kDelta * 4;         // identity blocks
constexpr uint32_t kBarBytes = 1024;
constexpr uint32_t kSmem = 1024 + kStages * kStageBytes + kA0Bytes + kHBytes + kBarBytes + kHistMax * 4;
static_assert(kSmem <= 232448, "shared memory budget");
}  // namespace dtc

// No-swizzle K-major core layout of one K = 8 TF32 operand (128 rows):
// [2 K halves][128 rows][16 B]  (LBO = 2048, SBO = 128).
__device__ __forceinline__ uint32_t dtc_none_off(int row, int u) {
  return (uint32_t)((u >> 2) * 2048 + row * 16 + (u & 3) * 4);
}

__global__ void __launch_bounds__(dtc::kThreads, 1)
assign_delta_tc_kernel(const __grid_constant__ CUtensorMap tm_qhi, const __grid_constant__ CUtensorMap tm_qlo,
                       const __grid_constant__ CUtensorMap tm_q0hi, const __grid_constant__ CUtensorMap tm_q0lo,
                       const __grid_constant__ CUtensorMap tm_fhi, const __grid_constant__ CUtensorMap tm_flo,
                       const __grid_constant__ CUtensorMap tm_ghi, const __grid_constant__ CUtensorMap tm_glo,
                       int64_t n, int d, int k, const int32_t* __restrict__ labels_prev,
                       int32_t* __restrict__ labels, float* __restrict__ mind, double* __restrict__ acc,
                       const long long* __restrict__ state) {
  using namespace dtc;
  if (stopped(state)) return;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw & 1023u)) & 1023u);
  uint8_t* sA0 = smem + kStages * kStageBytes;
  uint8_t* sH = sA0 + kA0Bytes;
  uint8_t* bar_area = sH + kHBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(bar_area);
  uint64_t* empty = full + kStages;
  uint64_t* a0full = empty + kStages;
  uint64_t* a0empty = a0full + 1;
  uint64_t* t0full = a0empty + 1;
  uint64_t* t0empty = t0full + 2;
  uint64_t* tbfull = t0empty + 2;
  uint64_t* tbempty = tbfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tbempty + 2);
  int* hist = reinterpret_cast<int*>(bar_area + kBarBytes);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool use_hist = acc != nullptr && k <= kHistMax;
  if (use_hist)
    for (int j = threadIdx.x; j < k; j += blockDim.x) hist[j] = 0;
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tm_qhi);
    ptx::prefetch_tmap(&tm_qlo);
    ptx::prefetch_tmap(&tm_fhi);
    ptx::prefetch_tmap(&tm_flo);
    ptx::prefetch_tmap(&tm_ghi);
    ptx::prefetch_tmap(&tm_glo);
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1 + 4);  // MMA commit + the 4 epilogue warps
    }
    ptx::mbar_init(a0full, 1);
    ptx::mbar_init(a0empty, 4);
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&t0full[b], 1);
      ptx::mbar_init(&t0empty[b], 4);
      ptx::mbar_init(&tbfull[b], 1);
      ptx::mbar_init(&tbempty[b], 4);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<512>(tmem_slot);
  if (warp == 3) {
    // H: 16 copies (one per centroid of the group) of the delta x delta identity
    for (int e = lane; e < kBN * kDelta; e += 32) {
      const int row = e / kDelta, u = e % kDelta;
      *reinterpret_cast<float*>(sH + dtc_none_off(row, u)) = (u == (row & (kDelta - 1))) ? 1.0f : 0.0f;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int64_t mtiles = (n + kBM - 1) / kBM;
  const int groups = (k + kNc - 1) / kNc;
  const int nb = (d + 1 + kDelta - 1) / kDelta;          // blocks carrying data (Delta r)
  const int nkc = (nb + 3) / 4;                           // 4 blocks per chunk

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    const uint64_t pol_b = ptx::policy_evict_last();
    const uint64_t pol_a = ptx::policy_evict_first();
    int stage = 0;
    uint32_t phase = 0, a0phase = 0;
    for (int64_t mt = blockIdx.x; mt < mtiles; mt += gridDim.x) {
      const int y_a = (int)(mt * kBM);
      ptx::mbar_wait(a0empty, a0phase ^ 1u);
      if (ptx::elect_one()) {
        ptx::mbar_expect_tx(a0full, kA0Bytes);
        ptx::tma_load_2d(&tm_q0hi, a0full, sA0, 0, y_a, pol_b);
        ptx::tma_load_2d(&tm_q0hi, a0full, sA0 + 2048, 4, y_a, pol_b);
        ptx::tma_load_2d(&tm_q0lo, a0full, sA0 + 4096, 0, y_a, pol_b);
        ptx::tma_load_2d(&tm_q0lo, a0full, sA0 + 6144, 4, y_a, pol_b);
      }
      __syncwarp();
      a0phase ^= 1u;
      for (int g = 0; g < groups; ++g) {
        const uint64_t pa = (g + 1 == groups) ? pol_a : pol_b;
        for (int kc = 0; kc < nkc; ++kc) {
          ptx::mbar_wait(&empty[stage], phase ^ 1u);
          uint8_t* st = smem + stage * kStageBytes;
          if (ptx::elect_one()) {
            ptx::mbar_expect_tx(&full[stage], kStageBytes);
            ptx::tma_load_2d(&tm_qhi, &full[stage], st, kc * kChunk, y_a, pa);
            ptx::tma_load_2d(&tm_qlo, &full[stage], st + kTile, kc * kChunk, y_a, pa);
            ptx::tma_load_2d(&tm_fhi, &full[stage], st + 2 * kTile, kc * kChunk, g * kBN, pol_b);
            ptx::tma_load_2d(&tm_flo, &full[stage], st + 3 * kTile, kc * kChunk, g * kBN, pol_b);
            ptx::tma_load_2d(&tm_ghi, &full[stage], st + 4 * kTile, kc * kChunk, g * kBN, pol_b);
            ptx::tma_load_2d(&tm_glo, &full[stage], st + 5 * kTile, kc * kChunk, g * kBN, pol_b);
          }
          __syncwarp();
          if (++stage == kStages) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t idesc = ptx::idesc_tf32<kBM, kBN>();
    const uint64_t q0hi = ptx::sdesc_k_none(ptx::smem_u32(sA0), 2048, 128);
    const uint64_t q0lo = ptx::sdesc_k_none(ptx::smem_u32(sA0 + 4096), 2048, 128);
    const uint64_t hd = ptx::sdesc_k_none(ptx::smem_u32(sH), 2048, 128);
    int stage = 0;
    uint32_t phase = 0, a0phase = 0;
    int t0b = 0, tbb = 0;
    uint32_t t0ph = 0, tbph = 0;
    for (int64_t mt = blockIdx.x; mt < mtiles; mt += gridDim.x) {
      ptx::mbar_wait(a0full, a0phase);
      a0phase ^= 1u;
      ptx::tc_fence_after();
      for (int g = 0; g < groups; ++g) {
        ptx::mbar_wait(&t0empty[t0b], t0ph ^ 1u);
        ptx::tc_fence_after();
        const uint32_t t0 = tmem + (uint32_t)(t0b * kBN);
        for (int kc = 0; kc < nkc; ++kc) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t base = ptx::smem_u32(smem + stage * kStageBytes);
          const uint64_t ahi = ptx::sdesc_k_sw128(base), alo = ptx::sdesc_k_sw128(base + kTile);
          const uint64_t fhi = ptx::sdesc_k_sw128(base + 2 * kTile), flo = ptx::sdesc_k_sw128(base + 3 * kTile);
          const uint64_t ghi = ptx::sdesc_k_sw128(base + 4 * kTile), glo = ptx::sdesc_k_sw128(base + 5 * kTile);
          for (int s = 0; s < 4; ++s) {
            const int b = kc * 4 + s;
            if (b >= nb) break;
            const uint64_t off = (uint64_t)(s * kDelta * 4) >> 4;  // 32 bytes per block
            if (b > 0) {
              ptx::mbar_wait(&tbempty[tbb], tbph ^ 1u);
              ptx::tc_fence_after();
            }
            if (ptx::elect_one()) {
              // T_0 += Q_b C_b0
              ptx::umma_tf32(t0, ahi + off, fhi + off, idesc, b != 0);
              ptx::umma_tf32(t0, ahi + off, flo + off, idesc, 1u);
              ptx::umma_tf32(t0, alo + off, fhi + off, idesc, 1u);
              if (b > 0) {
                // T_b = Q_0 C_0b + Q_b C_bb
                const uint32_t tb = tmem + (uint32_t)(2 * kBN + tbb * kBN);
                ptx::umma_tf32(tb, q0hi, ghi + off, idesc, 0u);
                ptx::umma_tf32(tb, q0hi, glo + off, idesc, 1u);
                ptx::umma_tf32(tb, q0lo, ghi + off, idesc, 1u);
                ptx::umma_tf32(tb, ahi + off, hd, idesc, 1u);
                ptx::umma_tf32(tb, alo + off, hd, idesc, 1u);
                ptx::umma_commit(&tbfull[tbb]);
              }
            }
            __syncwarp();
            if (b > 0) {
              tbb ^= 1;
              if (tbb == 0) tbph ^= 1u;
            }
          }
          if (ptx::elect_one()) ptx::umma_commit(&empty[stage]);
          __syncwarp();
          if (++stage == kStages) { stage = 0; phase ^= 1u; }
        }
        if (ptx::elect_one()) ptx::umma_commit(&t0full[t0b]);
        __syncwarp();
        t0b ^= 1;
        if (t0b == 0) t0ph ^= 1u;
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue ----------------
    const int ew = warp - 4;
    const int r = ew * 32 + lane;  // point within the tile = TMEM lane
    const uint32_t lane_base = (uint32_t)(ew * 32) << 16;
    int stage = 0;
    uint32_t phase = 0, a0phase = 0;
    int t0b = 0, tbb = 0;
    uint32_t t0ph = 0, tbph = 0;
    long long chg = 0;
    for (int64_t mt = blockIdx.x; mt < mtiles; mt += gridDim.x) {
      ptx::mbar_wait(a0full, a0phase);
      a0phase ^= 1u;
      float q0[kDelta];
#pragma unroll
      for (int u = 0; u < kDelta; ++u)
        q0[u] = *reinterpret_cast<const float*>(sA0 + dtc_none_off(r, u)) +
                *reinterpret_cast<const float*>(sA0 + 4096 + dtc_none_off(r, u));
      float best = INFINITY;
      int bj = 0;
      for (int g = 0; g < groups; ++g) {
        float D[kNc];
#pragma unroll
        for (int c = 0; c < kNc; ++c) D[c] = 0.0f;
        for (int kc = 0; kc < nkc; ++kc) {
          ptx::mbar_wait(&full[stage], phase);  // q_b of the stage is visible
          const uint8_t* st = smem + stage * kStageBytes;
          for (int s = 0; s < 4; ++s) {
            const int b = kc * 4 + s;
            if (b >= nb) break;
            if (b == 0) continue;
            // q_b = hi + lo (exact) from the 128B-swizzled A tile: 16-byte unit x of
            // row r sits at unit x ^ (r & 7)
            float q[kDelta];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint32_t o = (uint32_t)r * 128u + (uint32_t)(((2 * s + h) ^ (r & 7)) * 16);
              const float4 hi = *reinterpret_cast<const float4*>(st + o);
              const float4 lo = *reinterpret_cast<const float4*>(st + kTile + o);
              q[4 * h + 0] = hi.x + lo.x;
              q[4 * h + 1] = hi.y + lo.y;
              q[4 * h + 2] = hi.z + lo.z;
              q[4 * h + 3] = hi.w + lo.w;
            }
            ptx::mbar_wait(&tbfull[tbb], tbph);
            ptx::tc_fence_after();
            const uint32_t ta = tmem + lane_base + (uint32_t)(2 * kBN + tbb * kBN);
#pragma unroll
            for (int cb = 0; cb < kBN / 32; ++cb) {
              float v[32];
              ptx::tmem_ld_32x32b_x32(ta + cb * 32, v);
              if (cb == kBN / 32 - 1) {
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&tbempty[tbb]);
              }
#pragma unroll
              for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int u = 0; u < kDelta; ++u) D[cb * 4 + c] = fmaf(v[c * kDelta + u], q[u], D[cb * 4 + c]);
            }
            tbb ^= 1;
            if (tbb == 0) tbph ^= 1u;
          }
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&empty[stage]);
          if (++stage == kStages) { stage = 0; phase ^= 1u; }
        }
        ptx::mbar_wait(&t0full[t0b], t0ph);
        ptx::tc_fence_after();
        const uint32_t ta = tmem + lane_base + (uint32_t)(t0b * kBN);
#pragma unroll
        for (int cb = 0; cb < kBN / 32; ++cb) {
          float v[32];
          ptx::tmem_ld_32x32b_x32(ta + cb * 32, v);
          if (cb == kBN / 32 - 1) {
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&t0empty[t0b]);
          }
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int u = 0; u < kDelta; ++u) D[cb * 4 + c] = fmaf(v[c * kDelta + u], q0[u], D[cb * 4 + c]);
        }
        t0b ^= 1;
        if (t0b == 0) t0ph ^= 1u;
        // ascending centroid index, strict <: ties keep the lowest j (dense.py:56-68)
#pragma unroll
        for (int c = 0; c < kNc; ++c) {
          const int j = g * kNc + c;
          if (j < k && D[c] < best) { best = D[c]; bj = j; }
        }
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(a0empty);  // every MMA of the tile has completed (t0full)
      const int64_t row = mt * kBM + r;
      if (row < n) {
        labels[row] = bj;
        if (mind) mind[row] = best;
        if (acc) {
          if (labels_prev) chg += (labels_prev[row] != bj);
          if (use_hist) atomicAdd(&hist[bj], 1);
          else atomicAdd(&acc[(int64_t)k * d + bj], 1.0);
        }
        if (state != nullptr && !isfinite(best)) atomicExch((unsigned long long*)&state[kNanFlag], 1ull);
      }
    }
    if (acc) {
      chg = warp_sum(chg);
      if (lane == 0) atomicAdd(&acc[(int64_t)k * d + k + 1], (double)chg);
      ptx::named_bar_sync(1, 128);
      if (use_hist)
        for (int j = r; j < k; j += 128)
          if (hist[j]) atomicAdd(&acc[(int64_t)k * d + j], (double)hist[j]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc<512>(tmem);
}

// ---------------------------------------------------------------------------
// operand preparation
// ---------------------------------------------------------------------------
__device__ __forceinline__ float dtc_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Q = [1, p, 0...] (row stride ld), split into TF32 hi and the exact remainder lo.
__global__ void dtc_prep_points_kernel(const float* __restrict__ P, int64_t n, int d, int ld,
                                       float* __restrict__ qhi, float* __restrict__ qlo) {
  const int64_t total = n * (int64_t)ld;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / ld;
    const int c = (int)(e - i * ld);
    const float x = c == 0 ? 1.0f : (c <= d ? P[i * d + (c - 1)] : 0.0f);
    const float h = dtc_rna(x);
    qhi[e] = h;
    qlo[e] = x - h;
  }
}

// Entry (r, c) of centroid j's augmented matrix C_j = [[|c|^2, -c^T], [-c, I]]
// (zero outside the (d+1) x (d+1) corner: the padding of PAPER.md:154).
__device__ __forceinline__ float dtc_aug(const float* __restrict__ C, const float* __restrict__ cnorm, int j,
                                         int d, int r, int c) {
  if (r > d || c > d) return 0.0f;
  if (r == 0 && c == 0) return cnorm[j];
  if (r == 0) return -C[(int64_t)j * d + (c - 1)];
  if (c == 0) return -C[(int64_t)j * d + (r - 1)];
  return r == c ? 1.0f : 0.0f;
}

// F (row 8j+v, col 8b+u) = C_j[8b+u][v], G (row 8j+v, col 8b+u) = C_j[u][8b+v];
// rows of centroids j >= k are zero.  Split into TF32 hi / lo like Q.
__global__ void dtc_prep_centroids_kernel(const float* __restrict__ C, const float* __restrict__ cnorm, int k,
                                          int d, int ld, int rows, float* __restrict__ fhi,
                                          float* __restrict__ flo, float* __restrict__ ghi,
                                          float* __restrict__ glo) {
  const int64_t total = (int64_t)rows * ld;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(e / ld), col = (int)(e - (int64_t)row * ld);
    const int j = row / dtc::kDelta, v = row % dtc::kDelta;
    const int b = col / dtc::kDelta, u = col % dtc::kDelta;
    float f = 0.0f, g = 0.0f;
    if (j < k) {
      f = dtc_aug(C, cnorm, j, d, b * dtc::kDelta + u, v);
      g = dtc_aug(C, cnorm, j, d, u, b * dtc::kDelta + v);
    }
    const float fh = dtc_rna(f), gh = dtc_rna(g);
    fhi[e] = fh;
    flo[e] = f - fh;
    ghi[e] = gh;
    glo[e] = g - gh;
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 dtc_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (fn == nullptr) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// rows x ld f32, box = box_cols x 128 rows
static int dtc_tmap(CUtensorMap* m, const float* base, int64_t rows, int ld, int box_cols,
                    CUtensorMapSwizzle swz) {
  auto enc = dtc_encoder();
  if (!enc) return PCB_ENODEV;
  cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)dtc::kBM};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : PCB_EINVAL;
}

}  // namespace pcb

using namespace pcb;

extern "C" int pcb_delta_tc_ld(int d) { return (d + 1 + dtc::kChunk - 1) / dtc::kChunk * dtc::kChunk; }

extern "C" int pcb_delta_tc_kpad(int k) { return (k + dtc::kNc - 1) / dtc::kNc * dtc::kNc; }

extern "C" int pcb_delta_tc_prep_points(const float* P, int64_t n, int d, int ld, float* Q_hi, float* Q_lo,
                                        void* stream) {
  if (n < 1 || d < 1 || !P || !Q_hi || !Q_lo || ld != pcb_delta_tc_ld(d)) return PCB_EINVAL;
  const int64_t total = n * (int64_t)ld;
  const int grid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 16);
  dtc_prep_points_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(P, n, d, ld, Q_hi, Q_lo);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_delta_tc_prep_centroids(const float* C, const float* cnorm, int k, int d, int ld, float* F_hi,
                                           float* F_lo, float* G_hi, float* G_lo, void* stream) {
  if (k < 1 || d < 1 || !C || !cnorm || !F_hi || !F_lo || !G_hi || !G_lo || ld != pcb_delta_tc_ld(d))
    return PCB_EINVAL;
  const int rows = pcb_delta_tc_kpad(k) * dtc::kDelta;
  const int64_t total = (int64_t)rows * ld;
  const int grid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 16);
  dtc_prep_centroids_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(C, cnorm, k, d, ld, rows, F_hi, F_lo, G_hi,
                                                                     G_lo);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_assign_delta_tc_f32(const float* Q_hi, const float* Q_lo, int ld, int64_t n, int d,
                                       const float* F_hi, const float* F_lo, const float* G_hi, const float* G_lo,
                                       int k, const int32_t* labels_prev, int32_t* labels, float* mind,
                                       double* acc, const long long* state, void* stream) {
  if (n < 1 || d < 1 || k < 1 || !Q_hi || !Q_lo || !F_hi || !F_lo || !G_hi || !G_lo || !labels ||
      ld != pcb_delta_tc_ld(d))
    return PCB_EINVAL;
  if (n > INT32_MAX || (int64_t)pcb_delta_tc_kpad(k) * dtc::kDelta > INT32_MAX) return PCB_EUNSUP;
  const int brows = pcb_delta_tc_kpad(k) * dtc::kDelta;
  CUtensorMap tq_hi, tq_lo, tq0_hi, tq0_lo, tf_hi, tf_lo, tg_hi, tg_lo;
  int rc;
  if ((rc = dtc_tmap(&tq_hi, Q_hi, n, ld, dtc::kChunk, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
  if ((rc = dtc_tmap(&tq_lo, Q_lo, n, ld, dtc::kChunk, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
  if ((rc = dtc_tmap(&tq0_hi, Q_hi, n, ld, 4, CU_TENSOR_MAP_SWIZZLE_NONE))) return rc;
  if ((rc = dtc_tmap(&tq0_lo, Q_lo, n, ld, 4, CU_TENSOR_MAP_SWIZZLE_NONE))) return rc;
  if ((rc = dtc_tmap(&tf_hi, F_hi, brows, ld, dtc::kChunk, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
  if ((rc = dtc_tmap(&tf_lo, F_lo, brows, ld, dtc::kChunk, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
  if ((rc = dtc_tmap(&tg_hi, G_hi, brows, ld, dtc::kChunk, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
  if ((rc = dtc_tmap(&tg_lo, G_lo, brows, ld, dtc::kChunk, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
  cudaError_t e = cudaFuncSetAttribute(assign_delta_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)dtc::kSmem);
  if (e != cudaSuccess) return (int)e;
  const int64_t mtiles = (n + dtc::kBM - 1) / dtc::kBM;
  const int grid = (int)std::min<int64_t>(mtiles, (int64_t)sm_count());
  assign_delta_tc_kernel<<<grid, dtc::kThreads, dtc::kSmem, (cudaStream_t)stream>>>(
      tq_hi, tq_lo, tq0_hi, tq0_lo, tf_hi, tf_lo, tg_hi, tg_lo, n, d, k, labels_prev, labels, mind, acc, state);
  PCB_CHECK_LAUNCH();
  return 0;
}
