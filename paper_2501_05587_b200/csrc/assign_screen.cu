// Certified 1xTF32 screening for the distance stage (variant "tc1xtf32s").
//
// The 3xTF32 kernel (assign_tc.cu) runs at 95 % of the TF32 tensor pipe, so
// its only remaining lever is fewer tensor-core passes.  This kernel makes ONE
// TF32 pass over TF32-rounded operands p~ = rna(p), c~ = rna(c) (exactly
// representable, so the tensor core's f32->tf32 conversion is exact) and
// certifies the argmin with a rigorous error bound:
//
//   G  = <p, c>,  T = <p~, c~> (+ TC accumulation error)
//   |G - T| <= |da||c~| + |p~||dc| + |da||dc| + acc
//   (Cauchy-Schwarz on the exact residuals da = p - p~, dc = c - c~; acc is the
//   accumulation bound, 9 terms at 2^-23 per K=8 MMA)
//
// Ranking key  key_j = (cnorm_j + OFF) - 2 T_j,  OFF > max_i |p_i|^2 so keys are
// positive and can carry a 5-bit column index in their low mantissa bits
// (a single LOP3), making (value, index) min a plain FMNMX.  With a per-row
// uniform bound E_i (max over centroids of the B-side norms, plus every
// rounding of the key arithmetic and the packing), the true argmin j* obeys
// key_{j*} <= S1 + 2 E_i, so a row whose second-smallest key S2 exceeds
// S1 + 2 E_i has a certified, unique argmin.  Other rows ("ambiguous") are
// appended to a list and resolved by the 3xTF32 kernel on a compacted copy;
// their count is data dependent (~14 % right after a random-label init, ~3 %
// near convergence on the c3 blobs).
//
// Epilogue per accumulator element: the running min with its index uses
// 1 LOP3 + 0.5 FMNMX3 on the ALU pipe; the ambiguity test counts keys within
// 2E of the running min with saturating FFMAs (1 FFMA.SAT + 1 FADD on the FMA
// pipe), which is equivalent to the top-2 test (see the update rule in the
// chunk loop) at less than half the ALU work.
#include <cudaTypedefs.h>

#include "pcb_common.cuh"
#include "pcb_launch.cuh"
#include "tc_ptx.cuh"
#include "screen_common.cuh"

namespace pcb {

constexpr int SC_BM = 128;
constexpr int SC_THREADS = 384;  // warps 0-3 control, 4-11 epilogue (2 per TMEM lane group)

template <int BN>
struct ScCfg {
  static constexpr int kStages = BN == 256 ? 4 : 6;
  static constexpr uint32_t kABytes = SC_BM * SC_BK * 4;  // 16 KB
  static constexpr uint32_t kBBytes = BN * SC_BK * 4;
  static constexpr uint32_t kStageBytes = kABytes + kBBytes;
  static constexpr uint32_t kTmemCols = (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;
  static constexpr uint32_t kBarBytes = 4096;  // barriers, tmem slot, row-merge exchange (2 x 128 x 3 words)
  static constexpr uint32_t kSmem = 1024 + kStages * kStageBytes + kBarBytes + SC_KMAX * 4;
  static_assert(kSmem <= 232448, "exceeds the 227 KB dynamic shared memory limit");
};

// bstat layout (f32): [0] max_j |c~_j|, [1] max_j |dc_j|, [2] OFF, [3] spare
template <int BN>
__global__ void __launch_bounds__(SC_THREADS, 1)
assign_screen_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                     const float* __restrict__ anorm, const float* __restrict__ danorm,
                     const float* __restrict__ cnorm, const float* __restrict__ bstat, int64_t n, int k,
                     int num_kc, int32_t* __restrict__ labels, int* __restrict__ amb_list,
                     int* __restrict__ amb_count, const long long* __restrict__ state) {
  using Cfg = ScCfg<BN>;
  if (stopped(state)) return;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw & 1023u)) & 1023u);
  uint8_t* bar_area = smem + Cfg::kStages * Cfg::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(bar_area);
  uint64_t* empty = full + Cfg::kStages;
  uint64_t* tfull = empty + Cfg::kStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* xwritten = tempty + 2;    // [4 lane groups][2 slots]: h=1 published a slot
  uint64_t* xreleased = xwritten + 8; // [4][2]: h=0 consumed a slot
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xreleased + 8);
  float* cprime = reinterpret_cast<float*>(bar_area + Cfg::kBarBytes);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = (k + BN - 1) / BN;
  const float OFF = bstat[2];
  for (int j = threadIdx.x; j < ntiles * BN; j += blockDim.x)
    cprime[j] = j < k ? cnorm[j] + OFF : 3.0e38f;
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tm_a);
    ptx::prefetch_tmap(&tm_b);
    for (int s = 0; s < Cfg::kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], 256);
    }
    for (int b = 0; b < 8; ++b) {
      ptx::mbar_init(&xwritten[b], 32);
      ptx::mbar_init(&xreleased[b], 32);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t mtiles = (n + SC_BM - 1) / SC_BM;

  if (warp == 0) {
      const uint64_t pol_a = ptx::policy_evict_first();
      const uint64_t pol_b = ptx::policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t mt = blockIdx.x; mt < mtiles; mt += gridDim.x) {
        const int y_a = (int)(mt * SC_BM);
        for (int nt = 0; nt < ntiles; ++nt) {
          const uint64_t pa = (nt + 1 == ntiles) ? pol_a : pol_b;
          for (int kc = 0; kc < num_kc; ++kc) {
            ptx::mbar_wait(&empty[stage], phase ^ 1u);
            uint8_t* st = smem + stage * Cfg::kStageBytes;
            if (ptx::elect_one()) {
              ptx::mbar_expect_tx(&full[stage], Cfg::kStageBytes);
              ptx::tma_load_2d(&tm_a, &full[stage], st, kc * SC_BK, y_a, pa);
              ptx::tma_load_2d(&tm_b, &full[stage], st + Cfg::kABytes, kc * SC_BK, nt * BN, pol_b);
            }
            __syncwarp();
            if (++stage == Cfg::kStages) { stage = 0; phase ^= 1u; }
          }
        }
      }
    
  } else if (warp == 1) {
      constexpr uint32_t idesc = ptx::idesc_tf32<SC_BM, BN>();
      int stage = 0;
      uint32_t phase = 0;
      int abuf = 0;
      uint32_t aphase = 0;
      for (int64_t mt = blockIdx.x; mt < mtiles; mt += gridDim.x) {
        for (int nt = 0; nt < ntiles; ++nt) {
          ptx::mbar_wait(&tempty[abuf], aphase ^ 1u);
          ptx::tc_fence_after();
          const uint32_t dt = tmem + (uint32_t)(abuf * BN);
          for (int kc = 0; kc < num_kc; ++kc) {
            ptx::mbar_wait(&full[stage], phase);
            ptx::tc_fence_after();
            const uint32_t base = ptx::smem_u32(smem + stage * Cfg::kStageBytes);
            const uint64_t ad = ptx::sdesc_k_sw128(base);
            const uint64_t bd = ptx::sdesc_k_sw128(base + Cfg::kABytes);
if (ptx::elect_one()) {
#pragma unroll
              for (int ks = 0; ks < SC_BK / 8; ++ks) {
                const uint64_t off = (uint64_t)(ks * 8 * 4) >> 4;
                ptx::umma_tf32(dt, ad + off, bd + off, idesc, (kc | ks) != 0);
              }
              ptx::umma_commit(&empty[stage]);
            }
            __syncwarp();
            if (++stage == Cfg::kStages) { stage = 0; phase ^= 1u; }
          }
          if (ptx::elect_one()) ptx::umma_commit(&tfull[abuf]);
          __syncwarp();
          abuf ^= 1;
          if (abuf == 0) aphase ^= 1u;
        }
      }
    
  } else if (warp >= 4) {
    // Epilogue: warp w reads TMEM lane group (w % 4); the two warps of a group
    // (half h = 0/1) take alternating 32-column chunks and merge per row tile.
    const int g = warp & 3, h = (warp - 4) >> 2;
    const int r_in_tile = g * 32 + lane;
    float* xchg = reinterpret_cast<float*>(tmem_slot + 4);  // [2 slots][128][3]
    const float Bmax = bstat[0], dBmax = bstat[1];
    // TC accumulation: per K=8 MMA <= 9 terms aligned/truncated at 2^-23 of the
    // largest partial (|partial| <= sum |a~_t c~_t| <= |a~||c~|)
    const float acc_rel = (float)(num_kc * 4 + 2) * 9.0f * 0x1p-23f;
    const uint32_t msk = kIdxMask;
    int abuf = 0;
    uint32_t aphase = 0;
    int tile_it = 0;
    for (int64_t mt = blockIdx.x; mt < mtiles; mt += gridDim.x) {
      const int64_t row = mt * SC_BM + r_in_tile;
      // rigorous per-row bound on |key_j - OFF - s_j| (see header), rounded up
      float twoE = 0.0f;
      {
        const int64_t rr = row < n ? row : n - 1;
        const float an = anorm[rr], dan = danorm[rr];
        const float gerr = dan * Bmax + an * dBmax + dan * dBmax + acc_rel * an * Bmax;
        const float cbn = Bmax + dBmax;
        const float kmax = OFF + 2.0f * (an + dan) * cbn + cbn * cbn;
        twoE = 2.0f * 1.0001f * (2.0f * gerr + 0x1p-16f * kmax);
      }
      // counting scale: a key at least twoE/64 below the threshold counts 1
      const float big = 64.0f / twoE;
      // Running state: R1 = smallest packed key so far (index r1), cnt = number
      // of keys <= R1 + twoE (+margin), counted with saturating FFMAs on the
      // FMA pipe so the ALU pipe only carries the min (FMNMX3) and packing.
      float R1 = 3.4e38f, cnt = 0.0f;
      int r1 = 0;
      for (int nt = 0; nt < ntiles; ++nt) {
        ptx::mbar_wait(&tfull[abuf], aphase);
        ptx::tc_fence_after();
        const uint32_t taddr = tmem + ((uint32_t)(g * 32) << 16) + (uint32_t)(abuf * BN);
#pragma unroll 1
        for (int cb = h * 32; cb < BN; cb += 64) {
          float v[32];
          ptx::tmem_ld_32x32b_x32(taddr + cb, v);
          screen_chunk(v, cprime + nt * BN + cb, msk, nt * BN + cb, twoE, big, R1, r1, cnt);
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[abuf]);
        abuf ^= 1;
        if (abuf == 0) aphase ^= 1u;
      }
      // combine the two column halves of every row: h=1 publishes into a
      // double-buffered slot, h=0 consumes and releases it; mbarriers per lane
      // group and slot (phase = use count of the slot), so only the two warps
      // of a lane group ever wait on each other.
      const int sidx = tile_it & 1;
      const uint32_t use = (uint32_t)(tile_it >> 1);
      float* slot = xchg + sidx * (128 * 3);
      if (h == 1) {
        if (tile_it >= 2) ptx::mbar_wait(&xreleased[g * 2 + sidx], (use - 1u) & 1u);
        slot[r_in_tile * 3 + 0] = R1;
        slot[r_in_tile * 3 + 1] = cnt;
        slot[r_in_tile * 3 + 2] = __int_as_float(r1);
        ptx::mbar_arrive(&xwritten[g * 2 + sidx]);
      } else {
        ptx::mbar_wait(&xwritten[g * 2 + sidx], use & 1u);
        const float oR1 = slot[r_in_tile * 3 + 0], ocnt = slot[r_in_tile * 3 + 1];
        const int or1 = __float_as_int(slot[r_in_tile * 3 + 2]);
        ptx::mbar_arrive(&xreleased[g * 2 + sidx]);
        // each half certified its own candidates relative to its own min; the
        // row is unambiguous iff one half's min undercuts the other's by > 2E
        // and that half alone has a single candidate
        bool amb;
        if (oR1 < R1 - twoE) {
          amb = ocnt > 1.0f;
          R1 = oR1;
          r1 = or1;
        } else if (R1 < oR1 - twoE) {
          amb = cnt > 1.0f;
        } else {
          amb = true;
          if (oR1 < R1 || (oR1 == R1 && or1 < r1)) { R1 = oR1; r1 = or1; }
        }
        if (row < n) labels[row] = r1;
        amb = amb && row < n;
        const unsigned msk = __ballot_sync(0xffffffffu, amb);
        if (msk) {
          int base = 0;
          if (lane == 0) base = atomicAdd(amb_count, __popc(msk));
          base = __shfl_sync(0xffffffffu, base, 0);
          if (amb) amb_list[base + __popc(msk & ((1u << lane) - 1u))] = (int)row;
        }
      }
      ++tile_it;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc<Cfg::kTmemCols>(tmem);
}

// ---- screening prep / fallback helpers ---------------------------------------

__device__ __forceinline__ float rna_tf32(float x) {
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  return __uint_as_float(h);
}

__device__ __forceinline__ void atomic_max_pos(float* addr, float v) {
  atomicMax(reinterpret_cast<unsigned int*>(addr), __float_as_uint(v));  // v >= 0
}

// Per row of X (rows x d): |rna(x)|, |x - rna(x)| (rounded up), the max |x|^2,
// and optionally the rounded copy Xr (row stride ld, zero padded).
__global__ void __launch_bounds__(256)
row_tf32_norms_kernel(const float* __restrict__ X, int64_t rows, int d, float* __restrict__ an,
                      float* __restrict__ dan, float* __restrict__ maxsq, float* __restrict__ Xr, int ld) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float wmax = 0.0f;
  for (int64_t i = w; i < rows; i += nw) {
    double s_t = 0.0, s_d = 0.0, s_x = 0.0;
    if (Xr != nullptr)
      for (int t = d + lane; t < ld; t += 32) Xr[i * ld + t] = 0.0f;
    for (int t = lane; t < d; t += 32) {
      const float x = X[i * d + t];
      const float h = rna_tf32(x);
      if (Xr != nullptr) Xr[i * ld + t] = h;
      const double dd = (double)x - (double)h;
      s_t = fma((double)h, (double)h, s_t);
      s_d = fma(dd, dd, s_d);
      s_x = fma((double)x, (double)x, s_x);
    }
    s_t = warp_sum(s_t);
    s_d = warp_sum(s_d);
    s_x = warp_sum(s_x);
    if (lane == 0) {
      an[i] = (float)(sqrt(s_t) * (1.0 + 1e-6));
      dan[i] = (float)(sqrt(s_d) * (1.0 + 1e-6));
      wmax = fmaxf(wmax, (float)(s_x * (1.0 + 1e-6)));
    }
  }
  if (lane == 0 && maxsq != nullptr) atomic_max_pos(maxsq, wmax);
}

__global__ void max2_kernel(const float* __restrict__ b, const float* __restrict__ db, int k,
                            float* __restrict__ out) {
  float m0 = 0.0f, m1 = 0.0f;
  for (int j = threadIdx.x; j < k; j += blockDim.x) { m0 = fmaxf(m0, b[j]); m1 = fmaxf(m1, db[j]); }
  atomic_max_pos(&out[0], m0);
  atomic_max_pos(&out[1], m1);
}

__global__ void screen_stats_finish(float* __restrict__ bstat, const float* __restrict__ maxsq) {
  // OFF = 1.01 * max|p|^2 + 1 keeps every key positive
  bstat[2] = 1.01f * (*maxsq) + 1.0f;
}

// Gather the ambiguous rows into a compact TF32 hi/lo split (row stride ld).
__global__ void __launch_bounds__(256)
gather_split_rows(const float* __restrict__ P, int d, const int* __restrict__ list,
                  const int* __restrict__ count, int ld, float* __restrict__ hi, float* __restrict__ lo,
                  const long long* __restrict__ state) {
  if (stopped(state)) return;
  const int64_t cnt = *count;
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w; r < cnt; r += nw) {
    const int64_t i = list[r];
    for (int t = lane; t < ld; t += 32) {
      const float x = t < d ? P[i * d + t] : 0.0f;
      uint32_t h;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
      hi[r * ld + t] = __uint_as_float(h);
      lo[r * ld + t] = x - __uint_as_float(h);
    }
  }
}

__global__ void __launch_bounds__(256)
scatter_rows_labels(const int* __restrict__ list, const int* __restrict__ count,
                    const int32_t* __restrict__ sub, int32_t* __restrict__ labels,
                    const long long* __restrict__ state) {
  if (stopped(state)) return;
  const int64_t cnt = *count;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < cnt; r += (int64_t)gridDim.x * blockDim.x)
    labels[list[r]] = sub[r];
}

// counts and changed of the final labels (clustering.py:146-149) — used by the
// screened variant, whose assignment kernel only produces labels.
//
// With P and S (the delta update's persistent per-cluster f64 sums): when the
// previous iteration took the delta update (so this one most likely does too)
// the pass also applies the changed rows to S (S[new] += p, S[prev] -= p), the
// work of delta_sums_kernel, in the same stream over both label arrays;
// state[kSpec] tells pcb_update_mode, which then marks the mode 3 (delta sums
// done) or, if this iteration needs the full update, lets it overwrite S.
__global__ void __launch_bounds__(256)
count_labels_kernel(const int32_t* __restrict__ labels, const int32_t* __restrict__ prev, int64_t n, int k,
                    int d, double* __restrict__ acc, const long long* __restrict__ state,
                    const float* __restrict__ P = nullptr, double* __restrict__ S = nullptr) {
  if (stopped(state)) return;
  extern __shared__ int hist[];
  const AccLayout L{k, d};
  // every block reads the previous iteration's mode (nobody writes it before pcb_update_mode)
  const bool spec = S != nullptr && prev != nullptr && delta_mode(state);
  if (spec && blockIdx.x == 0 && threadIdx.x == 0) const_cast<long long*>(state)[kSpec] = 1;
  const int lane = threadIdx.x & 31;
  // changed rows of the warp's 32 x 4 labels, applied cooperatively (lanes over d)
  auto apply = [&](unsigned m, int64_t i0, int stride, int a, int b) {
    while (m) {
      const int src = __ffs(m) - 1;
      m &= m - 1;
      const int64_t r = i0 + (int64_t)src * stride;
      const int ja = __shfl_sync(0xffffffffu, a, src), jb = __shfl_sync(0xffffffffu, b, src);
      for (int t = lane; t < d; t += 32) {
        const double x = (double)P[r * d + t];
        atomicAdd(&S[(int64_t)jb * d + t], x);
        atomicAdd(&S[(int64_t)ja * d + t], -x);
      }
    }
  };
  for (int j = threadIdx.x; j < k; j += blockDim.x) hist[j] = 0;
  __syncthreads();
  long long chg = 0;
  // 16-byte loads (4 labels per thread and trip: the pass is a stream over
  // 8 bytes per row), scalar tail
  const bool al = ((reinterpret_cast<uintptr_t>(labels) | reinterpret_cast<uintptr_t>(prev)) & 15u) == 0;
  const int64_t n4 = al ? n >> 2 : 0;
  const int4* l4 = reinterpret_cast<const int4*>(labels);
  const int4* p4 = reinterpret_cast<const int4*>(prev);
  // warp-uniform trip counts (the changed-row ballots need the whole warp)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); i0 < n4; i0 += stride) {
    const int64_t i = i0 + lane;
    const bool in = i < n4;
    const int4 l = in ? l4[i] : make_int4(0, 0, 0, 0);
    if (in) {
      atomicAdd(&hist[l.x], 1);
      atomicAdd(&hist[l.y], 1);
      atomicAdd(&hist[l.z], 1);
      atomicAdd(&hist[l.w], 1);
    }
    if (prev) {
      const int4 q = in ? p4[i] : l;
      chg += (q.x != l.x) + (q.y != l.y) + (q.z != l.z) + (q.w != l.w);
      if (spec) {
        apply(__ballot_sync(0xffffffffu, q.x != l.x), 4 * i0 + 0, 4, q.x, l.x);
        apply(__ballot_sync(0xffffffffu, q.y != l.y), 4 * i0 + 1, 4, q.y, l.y);
        apply(__ballot_sync(0xffffffffu, q.z != l.z), 4 * i0 + 2, 4, q.z, l.z);
        apply(__ballot_sync(0xffffffffu, q.w != l.w), 4 * i0 + 3, 4, q.w, l.w);
      }
    }
  }
  for (int64_t i0 = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); i0 < n; i0 += stride) {
    const int64_t i = i0 + lane;
    const bool in = i < n;
    const int l = in ? labels[i] : 0;
    if (in) atomicAdd(&hist[l], 1);
    if (prev) {
      const int q = in ? prev[i] : l;
      chg += (q != l);
      if (spec) apply(__ballot_sync(0xffffffffu, q != l), i0, 1, q, l);
    }
  }
  chg = warp_sum(chg);
  if ((threadIdx.x & 31) == 0 && chg) atomicAdd(&acc[L.changed()], (double)chg);
  __syncthreads();
  for (int j = threadIdx.x; j < k; j += blockDim.x)
    if (hist[j]) atomicAdd(&acc[L.counts() + j], (double)hist[j]);
}

// large-k variant: global f64 atomics straight into acc
__global__ void count_labels_global_kernel(const int32_t* __restrict__ labels, const int32_t* __restrict__ prev,
                                           int64_t n, int k, int d, double* __restrict__ acc,
                                           const long long* __restrict__ state) {
  if (stopped(state)) return;
  const AccLayout L{k, d};
  long long chg = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int l = labels[i];
    atomicAdd(&acc[L.counts() + l], 1.0);
    if (prev) chg += (prev[i] != l);
  }
  chg = warp_sum(chg);
  if ((threadIdx.x & 31) == 0 && chg) atomicAdd(&acc[L.changed()], (double)chg);
}

template <int BN>
static int launch_screen(const float* P, int64_t n, int ld, const float* C, int k, const float* an,
                         const float* dan, const float* cnorm, const float* bstat, int32_t* labels,
                         int* amb_list, int* amb_count, const long long* state, cudaStream_t st) {
  using Cfg = ScCfg<BN>;
  CUtensorMap ta, tb;
  int rc;
  if ((rc = make_tmap_rows(&ta, P, n, ld, SC_BM))) return rc;
  if ((rc = make_tmap_rows(&tb, C, k, ld, BN))) return rc;
  auto kern = assign_screen_kernel<BN>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::kSmem);
  if (e != cudaSuccess) return (int)e;
  const int64_t mtiles = (n + SC_BM - 1) / SC_BM;
  const int grid = (int)std::min<int64_t>(mtiles, (int64_t)sm_count());
  kern<<<grid, SC_THREADS, Cfg::kSmem, st>>>(ta, tb, an, dan, cnorm, bstat, n, k, ld / SC_BK, labels,
                                             amb_list, amb_count, state);
  PCB_CHECK_LAUNCH();
  return 0;
}

}  // namespace pcb

using namespace pcb;

extern "C" int pcb_screen_prep_points(const float* P, int64_t n, int d, int ld, float* P_r, float* anorm,
                                      float* danorm, float* bstat, void* stream) {
  if (n < 1 || d < 1 || ld < d || ld % 32 || !P || !P_r || !anorm || !danorm || !bstat) return PCB_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(bstat, 0, 4 * sizeof(float), st);
  if (e != cudaSuccess) return (int)e;
  const int grid = (int)std::min<int64_t>((n * 32 + 255) / 256, (int64_t)sm_count() * 16);
  row_tf32_norms_kernel<<<grid, 256, 0, st>>>(P, n, d, anorm, danorm, bstat + 3, P_r, ld);
  PCB_CHECK_LAUNCH();
  screen_stats_finish<<<1, 1, 0, st>>>(bstat, bstat + 3);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_screen_prep_centroids(const float* C, int k, int d, float* bnorm, float* dbnorm,
                                         float* bstat, void* stream) {
  if (k < 1 || d < 1 || !C || !bnorm || !dbnorm || !bstat) return PCB_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(bstat, 0, 2 * sizeof(float), st);
  if (e != cudaSuccess) return (int)e;
  row_tf32_norms_kernel<<<(k * 32 + 255) / 256, 256, 0, st>>>(C, k, d, bnorm, dbnorm, nullptr, nullptr, 0);
  PCB_CHECK_LAUNCH();
  max2_kernel<<<1, 256, 0, st>>>(bnorm, dbnorm, k, bstat);  // bstat[0] = max|c~|, [1] = max|dc|
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_assign_screen_f32(const float* P_r, int64_t n, int ld, const float* C_r, int k,
                                     const float* cnorm, const float* anorm, const float* danorm,
                                     const float* bstat, int32_t* labels, int* amb_list, int* amb_count,
                                     const long long* state, void* stream) {
  if (n < 1 || ld < 32 || ld % 32 || k < 1 || !P_r || !C_r || !cnorm || !anorm || !danorm || !bstat || !labels ||
      !amb_list || !amb_count)
    return PCB_EINVAL;
  if (n > INT32_MAX) return PCB_EUNSUP;
  if (k > SC_KMAX) return PCB_EUNSUP;
  cudaStream_t st = (cudaStream_t)stream;
  if (k > 128)
    return launch_screen<256>(P_r, n, ld, C_r, k, anorm, danorm, cnorm, bstat, labels, amb_list, amb_count, state,
                              st);
  return launch_screen<128>(P_r, n, ld, C_r, k, anorm, danorm, cnorm, bstat, labels, amb_list, amb_count, state,
                            st);
}

extern "C" int pcb_resolve_ambiguous_f32(const float* P, int64_t n, int d, const int* amb_list,
                                         const int* amb_count, int ld, float* sub_hi, float* sub_lo,
                                         int32_t* sub_labels, const float* pnorm, const float* C,
                                         const float* C_hi, const float* C_lo, const float* cnorm, int k,
                                         int32_t* labels, int* flag_list, int* flag_count, void* scratch,
                                         int64_t scratch_bytes, const long long* state, void* stream) {
  if (n < 1 || d < 1 || k < 1 || ld < d || ld % 32 || !P || !amb_list || !amb_count || !sub_hi || !sub_lo ||
      !sub_labels || !pnorm || !C_hi || !C_lo || !cnorm || !labels ||
      (flag_list && (!flag_count || !C || !scratch || scratch_bytes < exact_scratch_bytes())))
    return PCB_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = sm_count() * 8;
  if (flag_list != nullptr) {
    cudaError_t e = cudaMemsetAsync(flag_count, 0, sizeof(int), st);
    if (e != cudaSuccess) return (int)e;
  }
  gather_split_rows<<<grid, 256, 0, st>>>(P, d, amb_list, amb_count, ld, sub_hi, sub_lo, state);
  PCB_CHECK_LAUNCH();
  int rc = assign_tc3xtf32_devcount(sub_hi, sub_lo, ld, pnorm, n, d, C_hi, C_lo, cnorm, k, sub_labels, amb_count,
                                    state, st, amb_list, flag_list, flag_count);
  if (rc) return rc;
  if (flag_list != nullptr &&
      (rc = exact_rows(P, d, C, k, flag_list, flag_count, amb_list, sub_labels, scratch, state, st)))
    return rc;
  scatter_rows_labels<<<grid, 256, 0, st>>>(amb_list, amb_count, sub_labels, labels, state);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int64_t pcb_exact_scratch_bytes(void) { return exact_scratch_bytes(); }

extern "C" int pcb_count_labels_delta_f32(const int32_t* labels, const int32_t* labels_prev, int64_t n, int k,
                                          int d, double* acc, const long long* state, const float* P, double* S,
                                          void* stream) {
  if (n < 1 || k < 1 || !labels || !labels_prev || !acc || !state || !P || !S) return PCB_EINVAL;
  if (k > 12288) return pcb_count_labels(labels, labels_prev, n, k, d, acc, state, stream);
  const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 4);
  count_labels_kernel<<<grid, 256, k * sizeof(int), (cudaStream_t)stream>>>(labels, labels_prev, n, k, d, acc,
                                                                          state, P, S);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_count_labels(const int32_t* labels, const int32_t* labels_prev, int64_t n, int k, int d,
                                double* acc, const long long* state, void* stream) {
  if (n < 1 || k < 1 || !labels || !acc) return PCB_EINVAL;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 4);
  if (k > 12288) {
    count_labels_global_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(labels, labels_prev, n, k, d, acc, state);
    PCB_CHECK_LAUNCH();
    return 0;
  }
  count_labels_kernel<<<grid, 256, k * sizeof(int), (cudaStream_t)stream>>>(labels, labels_prev, n, k, d, acc,
                                                                          state);
  PCB_CHECK_LAUNCH();
  return 0;
}
