// FFMA (CUDA-core) assignment kernels: distance + row argmin + bookkeeping.
//
// Replaces, for one Lloyd iteration, the reference's
//   D = pn[:,None] - 2.0*(P @ C.T) + cn[None,:]        clustering.py:310-311
//   raw = row_argmin(D)                                dense.py:56-68
//   counts / objective / changed bookkeeping           clustering.py:146-149
// without ever materialising the n x k matrix D.
//
// Distances are ranked on s_ij = cnorm_j - 2 <p_i, c_j> (the per-row constant
// pnorm_i does not change the argmin, dense.py's row-shift invariance), and the
// own distance mind_i = pnorm_i + s_i,label is what the objective sums.
// Ties break to the lowest centroid index (strict '<' in ascending j, and
// (v, j) lexicographic merges across threads).
//
// Two variants:
//  * assign_rowreg<T, DP, PPT>: one point per thread (PPT points), point held in
//    registers (d <= DP <= 32), centroids broadcast from shared memory.  This is
//    the small-d path of the north star (C1 d=2, C2 d=16).
//  * assign_tiled<T>: register-tiled SIMT GEMM (64x64x16 tiles, 4x4 per thread)
//    with the argmin fused in the epilogue; any d.  Used for f64 and as the
//    non-tensor-core fallback for large d.
#include <cstdlib>

#include "pcb_common.cuh"
#include "pcb_launch.cuh"

namespace pcb {

constexpr int kHistMax = 12288;  // per-block smem histogram (48 KB of int)

// Per-block bookkeeping shared by all assignment kernels: counts histogram and
// changed (labels != previous labels).  The objective is summed by the update
// kernel from exact own distances (see update.cu).
struct BlockBook {
  int* hist;        // smem, k ints, or nullptr -> direct global REDs
  long long changed;
};

__device__ __forceinline__ void book_point(BlockBook& b, double* acc, const AccLayout& L,
                                           int lab, const int32_t* labels_prev, int64_t i) {
  if (labels_prev != nullptr) b.changed += (labels_prev[i] != lab);
  if (b.hist != nullptr) atomicAdd(&b.hist[lab], 1);
  else atomicAdd(&acc[L.counts() + lab], 1.0);
}

__device__ void book_flush(BlockBook& b, double* acc, const AccLayout& L, int k) {
  __shared__ long long s_chg[32];
  long long c = warp_sum(b.changed);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) s_chg[w] = c;
  __syncthreads();
  if (w == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    c = lane < nw ? s_chg[lane] : 0;
    c = warp_sum(c);
    if (lane == 0) atomicAdd(&acc[L.changed()], (double)c);
  }
  if (b.hist != nullptr) {
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
      int h = b.hist[j];
      if (h) atomicAdd(&acc[L.counts() + j], (double)h);
    }
  }
}

__device__ __forceinline__ void flag_nonfinite(const long long* state, double v) {
  if (state != nullptr && !isfinite(v)) atomicExch((unsigned long long*)&state[kNanFlag], 1ull);
}

// ---------------------------------------------------------------------------
// Small-d: one point per thread, centroids in shared memory.
// ---------------------------------------------------------------------------
template <typename T, int DP, int PPT>
__global__ void __launch_bounds__(256)
assign_rowreg(const T* __restrict__ P, const T* __restrict__ pnorm, int64_t n, int d,
              const T* __restrict__ C, const T* __restrict__ cnorm, int k, int kc,
              const int32_t* __restrict__ labels_prev, int32_t* __restrict__ labels,
              T* __restrict__ mind, double* __restrict__ acc, const long long* __restrict__ state) {
  if (stopped(state)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sC = reinterpret_cast<T*>(smem_raw);          // [kc][DP]
  T* sN = sC + (size_t)kc * DP;                     // [kc]
  int* hist = reinterpret_cast<int*>(sN + kc);      // [k] (optional)
  const AccLayout L{k, d};
  BlockBook book{(acc != nullptr && k <= kHistMax) ? hist : nullptr, 0};
  if (book.hist) for (int j = threadIdx.x; j < k; j += blockDim.x) hist[j] = 0;

  auto load_chunk = [&](int c0) {
    const int cnt = min(kc, k - c0);
    for (int e = threadIdx.x; e < cnt * DP; e += blockDim.x) {
      const int jj = e / DP, t = e - jj * DP;
      sC[e] = t < d ? C[(int64_t)(c0 + jj) * d + t] : T(0);
    }
    for (int jj = threadIdx.x; jj < cnt; jj += blockDim.x) sN[jj] = cnorm[c0 + jj];
  };
  const bool single_chunk = (k <= kc);
  if (single_chunk) load_chunk(0);
  __syncthreads();

  const int64_t group = (int64_t)blockDim.x * PPT;
  for (int64_t base = (int64_t)blockIdx.x * group; base < n; base += (int64_t)gridDim.x * group) {
    T p[PPT][DP];
    int64_t idx[PPT];
#pragma unroll
    for (int r = 0; r < PPT; ++r) {
      idx[r] = base + threadIdx.x + (int64_t)r * blockDim.x;
      const int64_t ii = idx[r] < n ? idx[r] : (n - 1);
#pragma unroll
      for (int t = 0; t < DP; ++t) p[r][t] = t < d ? P[ii * d + t] : T(0);
    }
    T bv[PPT];
    int bj[PPT];
#pragma unroll
    for (int r = 0; r < PPT; ++r) { bv[r] = T(INFINITY); bj[r] = 0; }

    for (int c0 = 0; c0 < k; c0 += kc) {
      if (!single_chunk) { __syncthreads(); load_chunk(c0); __syncthreads(); }
      const int cnt = min(kc, k - c0);
      for (int jj = 0; jj < cnt; ++jj) {
        T c[DP];
#pragma unroll
        for (int t = 0; t < DP; ++t) c[t] = sC[jj * DP + t];
        const T cn = sN[jj];
#pragma unroll
        for (int r = 0; r < PPT; ++r) {
          T dot = T(0);
#pragma unroll
          for (int t = 0; t < DP; ++t) dot = fma(p[r][t], c[t], dot);
          const T s = fma(T(-2), dot, cn);
          if (s < bv[r]) { bv[r] = s; bj[r] = c0 + jj; }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < PPT; ++r) {
      if (idx[r] < n) {
        const T own = pnorm[idx[r]] + bv[r];
        labels[idx[r]] = bj[r];
        if (mind) mind[idx[r]] = own;
        if (acc) book_point(book, acc, L, bj[r], labels_prev, idx[r]);
        flag_nonfinite(state, (double)own);
      }
    }
  }
  if (acc) {
    __syncthreads();
    book_flush(book, acc, L, k);
  }
}

// ---------------------------------------------------------------------------
// Any d: register-tiled SIMT GEMM with fused argmin.  Block tile 64 points x
// 64 centroids x 16 dims, 256 threads, each thread a 4x4 micro-tile with rows
// ty+16r and columns tx+16c.  Every CTA walks all k centroids for its row
// tile, keeping a per-row running (value, index) minimum in registers.
// ---------------------------------------------------------------------------
constexpr int TBM = 64, TBN = 64, TBK = 16;

template <typename T>
__global__ void __launch_bounds__(256)
assign_tiled(const T* __restrict__ P, const T* __restrict__ pnorm, int64_t n, int d,
             const T* __restrict__ C, const T* __restrict__ cnorm, int k,
             const int32_t* __restrict__ labels_prev, int32_t* __restrict__ labels,
             T* __restrict__ mind, double* __restrict__ acc, const long long* __restrict__ state) {
  if (stopped(state)) return;
  __shared__ T As[TBK][TBM + 1];
  __shared__ T Bs[TBK][TBN + 1];
  __shared__ T sN[TBN];
  __shared__ int hist_s[kHistMax > 4096 ? 4096 : kHistMax];
  const AccLayout L{k, d};
  BlockBook book{(acc != nullptr && k <= 4096) ? hist_s : nullptr, 0};
  if (book.hist) for (int j = threadIdx.x; j < k; j += blockDim.x) hist_s[j] = 0;
  __syncthreads();

  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t mtiles = (n + TBM - 1) / TBM;
  for (int64_t mt = blockIdx.x; mt < mtiles; mt += gridDim.x) {
    const int64_t row0 = mt * TBM;
    T bv[4];
    int bj[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) { bv[r] = T(INFINITY); bj[r] = 0; }
    for (int col0 = 0; col0 < k; col0 += TBN) {
      T accm[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) accm[r][c] = T(0);
      for (int k0 = 0; k0 < d; k0 += TBK) {
        __syncthreads();
        for (int e = threadIdx.x; e < TBM * TBK; e += blockDim.x) {
          const int m = e / TBK, kk = e - m * TBK;
          const int64_t row = row0 + m;
          As[kk][m] = (row < n && k0 + kk < d) ? P[row * d + k0 + kk] : T(0);
          const int j = col0 + m;   // TBN == TBM
          Bs[kk][m] = (j < k && k0 + kk < d) ? C[(int64_t)j * d + k0 + kk] : T(0);
        }
        if (threadIdx.x < TBN) sN[threadIdx.x] = (col0 + threadIdx.x < k) ? cnorm[col0 + threadIdx.x] : T(0);
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < TBK; ++kk) {
          T a[4], b[4];
#pragma unroll
          for (int r = 0; r < 4; ++r) a[r] = As[kk][ty + 16 * r];
#pragma unroll
          for (int c = 0; c < 4; ++c) b[c] = Bs[kk][tx + 16 * c];
#pragma unroll
          for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) accm[r][c] = fma(a[r], b[c], accm[r][c]);
        }
      }
      // epilogue for this centroid tile: columns ascending within the thread
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int j = col0 + tx + 16 * c;
        if (j < k) {
          const T cn = sN[tx + 16 * c];
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const T s = fma(T(-2), accm[r][c], cn);
            argmin_merge(bv[r], bj[r], s, j);
          }
        }
      }
    }
    // merge across the 16 threads (tx) that share these rows
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) {
        T v2 = __shfl_xor_sync(0xffffffffu, bv[r], o);
        int j2 = __shfl_xor_sync(0xffffffffu, bj[r], o);
        argmin_merge(bv[r], bj[r], v2, j2);
      }
      const int64_t row = row0 + ty + 16 * r;
      if (tx == 0 && row < n) {
        const T own = pnorm[row] + bv[r];
        labels[row] = bj[r];
        if (mind) mind[row] = own;
        if (acc) book_point(book, acc, L, bj[r], labels_prev, row);
        flag_nonfinite(state, (double)own);
      }
    }
  }
  if (acc) {
    __syncthreads();
    book_flush(book, acc, L, k);
  }
}

// ---------------------------------------------------------------------------
// Small-d f32, packed: the same per-pair arithmetic as assign_rowreg (dot =
// fma over t in order, s = fma(-2, dot, cnorm), strict '<' in ascending j), two
// points per f32x2 register pair so that every FFMA2 advances two dot
// products.  Each thread holds NPAIR point pairs (2 NPAIR points) and walks the
// centroids two at a time (4 NPAIR independent FMA chains); centroid values
// come from shared memory duplicated as (c, c) pairs, so one LDS.128 feeds
// two k-steps of every pair.  Results are bit-identical to assign_rowreg.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long rp_pack(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void rp_unpack(unsigned long long r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ unsigned long long rp_ffma2(unsigned long long a, unsigned long long b,
                                                       unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

template <int DP, int NPAIR, int CJ>
__global__ void __launch_bounds__(256)
assign_rowpair(const float* __restrict__ P, const float* __restrict__ pnorm, int64_t n, int d,
               const float* __restrict__ C, const float* __restrict__ cnorm, int k, int kc,
               const int32_t* __restrict__ labels_prev, int32_t* __restrict__ labels,
               float* __restrict__ mind, double* __restrict__ acc, const long long* __restrict__ state) {
  if (stopped(state)) return;
  constexpr int PPT = 2 * NPAIR;
  constexpr int SPR = DP + 1;                                // padded row stride of the point stage
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* sC = reinterpret_cast<float2*>(smem_raw);          // [kc2][DP] (c, c) pairs
  const int kc2 = (kc + CJ - 1) / CJ * CJ;                   // centroids in steps of CJ
  float* sN = reinterpret_cast<float*>(sC + (size_t)kc2 * DP);  // [kc2]
  float* sP = sN + kc2;                                      // [warps][32][SPR] point stage
  int* hist = reinterpret_cast<int*>(sP + (blockDim.x >> 5) * 32 * SPR);
  const AccLayout L{k, d};
  BlockBook book{(acc != nullptr && k <= kHistMax) ? hist : nullptr, 0};
  if (book.hist) for (int j = threadIdx.x; j < k; j += blockDim.x) hist[j] = 0;

  auto load_chunk = [&](int c0) {
    const int cnt = min(kc, k - c0);
    for (int e = threadIdx.x; e < kc2 * DP; e += blockDim.x) {
      const int jj = e / DP, t = e - jj * DP;
      const float v = (jj < cnt && t < d) ? C[(int64_t)(c0 + jj) * d + t] : 0.0f;
      sC[e] = make_float2(v, v);
    }
    // padding centroids of a ragged chunk: s = +inf never beats a real key
    for (int jj = threadIdx.x; jj < kc2; jj += blockDim.x) sN[jj] = jj < cnt ? cnorm[c0 + jj] : INFINITY;
  };
  const bool single_chunk = (k <= kc);
  if (single_chunk) load_chunk(0);
  __syncthreads();

  const unsigned long long m2 = rp_pack(-2.0f, -2.0f);
  const int64_t group = (int64_t)blockDim.x * PPT;
  const int lane = threadIdx.x & 31;
  float* wP = sP + (threadIdx.x >> 5) * 32 * SPR;
  for (int64_t base = (int64_t)blockIdx.x * group; base < n; base += (int64_t)gridDim.x * group) {
    unsigned long long pp[NPAIR][DP];
    int64_t idx[PPT];
#pragma unroll
    for (int r = 0; r < PPT; ++r) idx[r] = base + threadIdx.x + (int64_t)r * blockDim.x;
    // per-row inputs of the epilogue, fetched now so their latency overlaps the distances
    float pn_r[PPT];
    int lp_r[PPT];
#pragma unroll
    for (int r = 0; r < PPT; ++r) {
      const int64_t ii = idx[r] < n ? idx[r] : n - 1;
      pn_r[r] = pnorm[ii];
      lp_r[r] = labels_prev != nullptr ? labels_prev[ii] : 0;
    }
    // The 32 rows of a warp for point slot r are contiguous in P: read them
    // coalesced (lane-strided over 32 d floats, every load of the round in
    // flight at once) into the warp's padded stage, then every lane takes its
    // own row (row-per-lane reads of P would cost one L1 wavefront per lane per
    // column).  (A register prefetch of the next round was tried: the extra
    // registers cost more occupancy than the hidden latency gained.)
    float tmp[PPT][DP];
#pragma unroll
    for (int r = 0; r < PPT; ++r) {
      const int64_t row0 = idx[r] - lane;
      const int64_t avail = n - row0 < 32 ? n - row0 : 32;  // rows of this warp slot inside P
      const float* src = P + row0 * d;
      const int lim = (int)avail * d;
#pragma unroll
      for (int i = 0; i < DP; ++i) {
        const int e = lane + 32 * i;
        tmp[r][i] = (i < d && e < lim) ? __ldg(src + e) : 0.0f;
      }
    }
    float pv[PPT][DP];
#pragma unroll
    for (int r = 0; r < PPT; ++r) {
      __syncwarp();
#pragma unroll
      for (int i = 0; i < DP; ++i) {
        const int e = lane + 32 * i;
        if (i < d) {
          const int rr = e / d, t = e - rr * d;
          wP[rr * SPR + t] = tmp[r][i];
        }
      }
      __syncwarp();
#pragma unroll
      for (int t = 0; t < DP; ++t) pv[r][t] = t < d ? wP[lane * SPR + t] : 0.0f;
    }
#pragma unroll
    for (int q = 0; q < NPAIR; ++q)
#pragma unroll
      for (int t = 0; t < DP; ++t) pp[q][t] = rp_pack(pv[2 * q][t], pv[2 * q + 1][t]);
    float bv[PPT];
    int bj[PPT];
#pragma unroll
    for (int r = 0; r < PPT; ++r) { bv[r] = INFINITY; bj[r] = 0; }

    for (int c0 = 0; c0 < k; c0 += kc) {
      if (!single_chunk) { __syncthreads(); load_chunk(c0); __syncthreads(); }
      const int cnt2 = (min(kc, k - c0) + CJ - 1) / CJ * CJ;
      for (int jj = 0; jj < cnt2; jj += CJ) {
        unsigned long long dot[NPAIR][CJ];
#pragma unroll
        for (int q = 0; q < NPAIR; ++q)
#pragma unroll
          for (int u = 0; u < CJ; ++u) dot[q][u] = 0ull;
#pragma unroll
        for (int t2 = 0; t2 < (DP + 1) / 2; ++t2) {
          float4 v[CJ];
#pragma unroll
          for (int u = 0; u < CJ; ++u) {
            if (DP == 1) {
              const float2 a1 = sC[(size_t)(jj + u) * DP];
              v[u] = make_float4(a1.x, a1.y, 0.0f, 0.0f);
            } else {
              v[u] = reinterpret_cast<const float4*>(sC + (size_t)(jj + u) * DP)[t2];
            }
          }
#pragma unroll
          for (int u = 0; u < CJ; ++u) {
            const unsigned long long c0v = rp_pack(v[u].x, v[u].y);
#pragma unroll
            for (int q = 0; q < NPAIR; ++q) dot[q][u] = rp_ffma2(pp[q][2 * t2], c0v, dot[q][u]);
          }
          if (2 * t2 + 1 < DP) {
#pragma unroll
            for (int u = 0; u < CJ; ++u) {
              const unsigned long long c1v = rp_pack(v[u].z, v[u].w);
#pragma unroll
              for (int q = 0; q < NPAIR; ++q) dot[q][u] = rp_ffma2(pp[q][2 * t2 + 1], c1v, dot[q][u]);
            }
          }
        }
        // keys and the running argmin in ascending centroid order (strict '<')
#pragma unroll
        for (int u = 0; u < CJ; ++u) {
          const unsigned long long nu = rp_pack(sN[jj + u], sN[jj + u]);
#pragma unroll
          for (int q = 0; q < NPAIR; ++q) {
            float s0, s1;
            rp_unpack(rp_ffma2(dot[q][u], m2, nu), s0, s1);  // centroid jj + u, points 2q, 2q + 1
            if (s0 < bv[2 * q]) { bv[2 * q] = s0; bj[2 * q] = c0 + jj + u; }
            if (s1 < bv[2 * q + 1]) { bv[2 * q + 1] = s1; bj[2 * q + 1] = c0 + jj + u; }
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < PPT; ++r) {
      if (idx[r] < n) {
        const float own = pn_r[r] + bv[r];
        labels[idx[r]] = bj[r];
        if (mind) mind[idx[r]] = own;
        if (acc) {
          if (labels_prev != nullptr) book.changed += (lp_r[r] != bj[r]);
          if (book.hist != nullptr) atomicAdd(&book.hist[bj[r]], 1);
          else atomicAdd(&acc[L.counts() + bj[r]], 1.0);
        }
        flag_nonfinite(state, (double)own);
      }
    }
  }
  if (acc) {
    __syncthreads();
    book_flush(book, acc, L, k);
  }
}

// ---------------------------------------------------------------------------
// assign_rowcst<D>: assign_rowpair's arithmetic (bit-identical labels / keys)
// with the centroids in the constant bank instead of shared memory, for
// d == D and k (D + 1) floats within the constant cache's 8 KB working set
// (c2: d=16, k=64).  ncu of the shared-memory kernels at c2 put a
// third of all warp stalls on the short scoreboard of the centroid LDS.128s;
// from the constant bank the compiler loads two centroid values per LDCU.64
// into uniform registers and FFMA2 takes each as a broadcast scalar operand
// (`FFMA2 R, R.F32x2, UR.F32, R`), so no vector register or shared-memory
// wavefront is spent on centroids and the loads hoist freely.  The centroids
// and their norms are copied into the bank (one D2D copy on the launching
// stream when the norms follow the centroid rows in memory, as the engine lays
// them out; graph-capturable) before each launch; the bank is one per process
// and device, so launches that use it must be ordered (one stream), as every
// launch of an engine is.
// ---------------------------------------------------------------------------
constexpr int kCstFloats = 2048;
__constant__ float c_cst[kCstFloats];

template <int D, int NPAIR, int U>
__device__ __forceinline__ void rc_block(const unsigned long long (&pp)[NPAIR][D], int jj, int k,
                                         float (&bv)[2 * NPAIR], int (&bj)[2 * NPAIR]) {
  const unsigned long long m2 = rp_pack(-2.0f, -2.0f);
  unsigned long long dot[NPAIR][U];
#pragma unroll
  for (int q = 0; q < NPAIR; ++q)
#pragma unroll
    for (int u = 0; u < U; ++u) dot[q][u] = 0ull;
#pragma unroll
  for (int t = 0; t < D; ++t) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float c = c_cst[(jj + u) * D + t];
      const unsigned long long cc = rp_pack(c, c);
#pragma unroll
      for (int q = 0; q < NPAIR; ++q) dot[q][u] = rp_ffma2(pp[q][t], cc, dot[q][u]);
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const float cn = c_cst[k * D + jj + u];
    const unsigned long long nu = rp_pack(cn, cn);
#pragma unroll
    for (int q = 0; q < NPAIR; ++q) {
      float s0, s1;
      rp_unpack(rp_ffma2(dot[q][u], m2, nu), s0, s1);
      if (s0 < bv[2 * q]) { bv[2 * q] = s0; bj[2 * q] = jj + u; }
      if (s1 < bv[2 * q + 1]) { bv[2 * q + 1] = s1; bj[2 * q + 1] = jj + u; }
    }
  }
}

__device__ __forceinline__ void rc_cp_async4(void* dst, const void* src, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(s), "l"(src), "r"(src_bytes) : "memory");
}

// Prefetch one group (1024 rows: slot r of warp w = the 32 contiguous rows
// base + 256 r + 32 w ..) into the warp's stage with cp.async, coalesced 4-byte
// copies (a warp reads 32 consecutive floats per copy), rows past n zero-filled.
// The stage holds the two points of each lane's pair q (slots 2q, 2q + 1)
// interleaved: 16-byte chunk c of lane-row r = (a_2c, b_2c, a_2c+1, b_2c+1), so
// one LDS.128 yields two packed f32x2 operands and no register ever packs a
// pair (a packing MOV is cheap enough that ptxas rematerialises it inside the
// centroid loop: 220 IMAD.MOVs per 136 FFMA2s).  Chunk c of lane-row r sits at
// (c + r / R) mod CH (CH = chunks per lane-row, R = lane-rows per 128-byte
// line): the row-per-lane LDS.128s are conflict-free.
template <int D>
__device__ __forceinline__ void rc_prefetch(const float* __restrict__ P, int64_t n, int64_t base, float* stage) {
  constexpr int CH = D / 2, R = 8 / CH, RS = 32 / D;   // RS: rows per 32 consecutive floats
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int t = lane % D, r0 = lane / D;                 // copy i of a slot: row r0 + RS i, column t
  float* dl = stage + (t & 1) * 2;
#pragma unroll
  for (int sl = 0; sl < 4; ++sl) {
    const int64_t rb = base + 256 * sl + 32 * w;
    float* dq = dl + (sl >> 1) * (32 * 2 * D) + (sl & 1);
    const float* src = P + (rb + r0) * D + t;
    if (rb + 32 <= n) {
#pragma unroll
      for (int i = 0; i < D; ++i) {
        const int row = r0 + RS * i;
        rc_cp_async4(dq + row * 2 * D + (((t >> 1) + row / R) % CH) * 4, src + (int64_t)RS * i * D, 4);
      }
    } else {
#pragma unroll
      for (int i = 0; i < D; ++i) {
        const int row = r0 + RS * i;
        const bool in = rb + row < n;
        rc_cp_async4(dq + row * 2 * D + (((t >> 1) + row / R) % CH) * 4, in ? src + (int64_t)RS * i * D : P,
                     in ? 4 : 0);
      }
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// Persistent loop over 1024-row groups; each warp's next group streams into its
// stage (cp.async) while it computes the current one, so the per-group load
// (every warp of the GPU loading at once, ~19 MB per wave at c2) no longer
// idles the FMA pipe.  (Measured: 58.3 -> 57.5 us at c2; most of the gain over
// the shared-memory kernel is the constant bank.)
template <int D>
__global__ void __launch_bounds__(256, 2)
assign_rowcst(const float* __restrict__ P, const float* __restrict__ pnorm, int64_t n, int k,
              const int32_t* __restrict__ labels_prev, int32_t* __restrict__ labels,
              float* __restrict__ mind, double* __restrict__ acc, const long long* __restrict__ state,
              double* __restrict__ S) {
  if (stopped(state)) return;
  // With S (the delta update's persistent per-cluster f64 sums) and the
  // previous iteration a delta one: apply each changed row to S here, from the
  // point values already in registers (S[new] += p, S[prev] -= p), the work of
  // delta_sums_kernel; state[kSpec] tells pcb_update_mode (as the screen
  // path's count pass does, assign_screen.cu count_labels_kernel).
  const bool spec = S != nullptr && labels_prev != nullptr && acc != nullptr && delta_mode(state);
  if (spec && blockIdx.x == 0 && threadIdx.x == 0) const_cast<long long*>(state)[kSpec] = 1;
  constexpr int NPAIR = 2, PPT = 4, CJ = 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* stage = reinterpret_cast<float*>(smem_raw) + (threadIdx.x >> 5) * (PPT * 32 * D);
  int* hist = reinterpret_cast<int*>(reinterpret_cast<float*>(smem_raw) + (blockDim.x >> 5) * (PPT * 32 * D));
  const AccLayout L{k, D};
  BlockBook book{(acc != nullptr && k <= kHistMax) ? hist : nullptr, 0};
  if (book.hist) for (int j = threadIdx.x; j < k; j += blockDim.x) hist[j] = 0;
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int64_t group = (int64_t)blockDim.x * PPT;
  const int64_t ng = (n + group - 1) / group;
  int64_t g = blockIdx.x;
  if (g < ng) rc_prefetch<D>(P, n, g * group, stage);
  for (; g < ng; g += gridDim.x) {
    const int64_t base = g * group;
    int64_t idx[PPT];
#pragma unroll
    for (int r = 0; r < PPT; ++r) idx[r] = base + threadIdx.x + (int64_t)r * blockDim.x;
    float pn_r[PPT];
    int lp_r[PPT];
#pragma unroll
    for (int r = 0; r < PPT; ++r) {
      const int64_t ii = idx[r] < n ? idx[r] : n - 1;
      pn_r[r] = pnorm[ii];
      lp_r[r] = labels_prev != nullptr ? labels_prev[ii] : 0;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    unsigned long long pp[NPAIR][D];
#pragma unroll
    for (int q = 0; q < NPAIR; ++q)
#pragma unroll
      for (int c = 0; c < D / 2; ++c) {
        const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(
            stage + q * (32 * 2 * D) + lane * 2 * D + ((c + lane / (16 / D)) % (D / 2)) * 4);
        pp[q][2 * c] = v.x;
        pp[q][2 * c + 1] = v.y;
      }
    __syncwarp();
    if (g + gridDim.x < ng) rc_prefetch<D>(P, n, (g + gridDim.x) * group, stage);

    float bv[PPT];
    int bj[PPT];
#pragma unroll
    for (int r = 0; r < PPT; ++r) { bv[r] = INFINITY; bj[r] = 0; }
    int jj = 0;
    for (; jj + CJ <= k; jj += CJ) rc_block<D, NPAIR, CJ>(pp, jj, k, bv, bj);
    for (; jj < k; ++jj) rc_block<D, NPAIR, 1>(pp, jj, k, bv, bj);
#pragma unroll
    for (int r = 0; r < PPT; ++r) {
      if (idx[r] < n) {
        const float own = pn_r[r] + bv[r];
        labels[idx[r]] = bj[r];
        if (mind) mind[idx[r]] = own;
        if (acc) {
          if (labels_prev != nullptr) book.changed += (lp_r[r] != bj[r]);
          if (book.hist != nullptr) atomicAdd(&book.hist[bj[r]], 1);
          else atomicAdd(&acc[L.counts() + bj[r]], 1.0);
        }
        flag_nonfinite(state, (double)own);
      }
    }
    if (spec) {
      // changed rows of the warp, one at a time with the lanes over the
      // columns (the row was just read: an L1/L2 hit), as delta_sums_kernel
      const int lane = threadIdx.x & 31;
#pragma unroll
      for (int r = 0; r < PPT; ++r) {
        unsigned m = __ballot_sync(0xffffffffu, idx[r] < n && lp_r[r] != bj[r]);
        while (m) {
          const int src = __ffs(m) - 1;
          m &= m - 1;
          const int ja = __shfl_sync(0xffffffffu, lp_r[r], src), jb = __shfl_sync(0xffffffffu, bj[r], src);
          const int64_t row = idx[r] - lane + src;
          if (lane < D) {
            const double x = (double)P[row * D + lane];
            atomicAdd(&S[(int64_t)jb * D + lane], x);
            atomicAdd(&S[(int64_t)ja * D + lane], -x);
          }
        }
      }
    }
  }
  if (acc) {
    __syncthreads();
    book_flush(book, acc, L, k);
  }
}

template <int D>
static int launch_rowcst(const float* P, const float* pnorm, int64_t n, const float* C, const float* cnorm, int k,
                         const int32_t* lp, int32_t* lab, float* mind, double* acc, const long long* state,
                         double* S, cudaStream_t st) {
  // the bank's device address and the smem opt-in are per device
  static float* banks[64] = {nullptr};
  static bool attrs[64] = {false};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return (int)e;
  if (dev < 0 || dev >= 64) return PCB_EUNSUP;
  if (banks[dev] == nullptr) {
    void* a = nullptr;
    e = cudaGetSymbolAddress(&a, c_cst);
    if (e != cudaSuccess) return (int)e;
    banks[dev] = static_cast<float*>(a);
  }
  float* bank = banks[dev];
  // one copy when the norms follow the centroid rows in memory (the engine's
  // layout), two otherwise
  if (cnorm == C + (size_t)k * D) {
    e = cudaMemcpyAsync(bank, C, (size_t)k * (D + 1) * sizeof(float), cudaMemcpyDeviceToDevice, st);
  } else {
    e = cudaMemcpyAsync(bank, C, (size_t)k * D * sizeof(float), cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(bank + (size_t)k * D, cnorm, (size_t)k * sizeof(float), cudaMemcpyDeviceToDevice, st);
  }
  if (e != cudaSuccess) return (int)e;
  const size_t smem = (size_t)8 * 4 * 32 * D * sizeof(float) +
                      ((acc != nullptr && k <= kHistMax) ? (size_t)k * sizeof(int) : 0);
  auto kern = assign_rowcst<D>;
  if (!attrs[dev]) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024 + kHistMax * 4);
    if (e != cudaSuccess) return (int)e;
    attrs[dev] = true;
  }
  const int64_t groups = (n + 256 * 4 - 1) / (256 * 4);
  const int grid = (int)std::min<int64_t>(groups, (int64_t)persistent_grid(kern, 256, smem));
  kern<<<grid, 256, smem, st>>>(P, pnorm, n, k, lp, lab, mind, acc, state, S);
  PCB_CHECK_LAUNCH();
  return 0;
}

// the constant-bank kernel serves d in {8, 16} when the centroids and norms fit
// the bank and P's rows are 16-byte aligned for cp.async (at c1's d = 2,
// k = 10 the launch is latency-bound and the bank copies cost more than they
// save: 8.8 vs 11.1 us); PCB_ROWCST_OFF selects the shared-memory kernel (A/B)
static bool rowcst_fits(const float* P, int d, int k) {
  static const bool off = getenv("PCB_ROWCST_OFF") != nullptr;
  return !off && (d == 8 || d == 16) && (int64_t)k * (d + 1) <= kCstFloats && ((uintptr_t)P & 15) == 0;
}

template <int DP, int NPAIR, int CJ = 2>
static int launch_rowpair(const float* P, const float* pnorm, int64_t n, int d, const float* C, const float* cnorm,
                          int k, const int32_t* lp, int32_t* lab, float* mind, double* acc, const long long* state,
                          cudaStream_t st) {
  const int per = (2 * DP + 1) * (int)sizeof(float);
  int kc = (32768 / per) & ~(CJ - 1);
  if (kc > k) kc = k;
  const int kc2 = (kc + CJ - 1) / CJ * CJ;
  size_t smem = (size_t)kc2 * per + (size_t)8 * 32 * (DP + 1) * sizeof(float) +
                ((acc != nullptr && k <= kHistMax) ? (size_t)k * sizeof(int) : 0);
  auto kern = assign_rowpair<DP, NPAIR, CJ>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
  }
  const int64_t groups = (n + 256 * 2 * NPAIR - 1) / (256 * 2 * NPAIR);
  const int grid = (int)std::min<int64_t>(groups, (int64_t)persistent_grid(kern, 256, smem));
  kern<<<grid, 256, smem, st>>>(P, pnorm, n, d, C, cnorm, k, kc, lp, lab, mind, acc, state);
  PCB_CHECK_LAUNCH();
  return 0;
}

template <typename T, int DP, int PPT>
static int launch_rowreg(const T* P, const T* pnorm, int64_t n, int d, const T* C, const T* cnorm,
                         int k, const int32_t* lp, int32_t* lab, T* mind, double* acc,
                         const long long* state, cudaStream_t st) {
  const int per = (DP + 1) * (int)sizeof(T);
  int kc = 32768 / per;
  if (kc > k) kc = k;
  size_t smem = (size_t)kc * per + ((acc != nullptr && k <= kHistMax) ? (size_t)k * sizeof(int) : 0);
  auto kern = assign_rowreg<T, DP, PPT>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
  }
  const int64_t groups = (n + 256 * PPT - 1) / (256 * PPT);
  const int grid = (int)std::min<int64_t>(groups, (int64_t)persistent_grid(kern, 256, smem));
  kern<<<grid, 256, smem, st>>>(P, pnorm, n, d, C, cnorm, k, kc, lp, lab, mind, acc, state);
  PCB_CHECK_LAUNCH();
  return 0;
}

template <typename T>
static int assign_dispatch(const T* P, const T* pnorm, int64_t n, int d, const T* C, const T* cnorm,
                           int k, const int32_t* lp, int32_t* lab, T* mind, double* acc,
                           const long long* state, int variant, cudaStream_t st, double* S = nullptr) {
  if (n < 1 || d < 1 || k < 1 || !P || !pnorm || !C || !cnorm || !lab) return PCB_EINVAL;
  if (variant == PCB_ASSIGN_AUTO) variant = (d <= 32) ? PCB_ASSIGN_ROWREG : PCB_ASSIGN_TILED;
  if (variant == PCB_ASSIGN_ROWREG && sizeof(T) == 4 && getenv("PCB_ROWREG_SCALAR") == nullptr) {
    // f32: packed two-points-per-FFMA2 kernel (bit-identical to assign_rowreg)
    const float* Pf = reinterpret_cast<const float*>(P);
    const float* pn = reinterpret_cast<const float*>(pnorm);
    const float* Cf = reinterpret_cast<const float*>(C);
    const float* cn = reinterpret_cast<const float*>(cnorm);
    float* md = reinterpret_cast<float*>(mind);
    if (rowcst_fits(Pf, d, k)) {
      if (d == 8) return launch_rowcst<8>(Pf, pn, n, Cf, cn, k, lp, lab, md, acc, state, S, st);
      return launch_rowcst<16>(Pf, pn, n, Cf, cn, k, lp, lab, md, acc, state, S, st);
    }
    if (d <= 1) return launch_rowpair<1, 2>(Pf, pn, n, d, Cf, cn, k, lp, lab, md, acc, state, st);
    if (d <= 2) return launch_rowpair<2, 2>(Pf, pn, n, d, Cf, cn, k, lp, lab, md, acc, state, st);
    if (d <= 4) return launch_rowpair<4, 2>(Pf, pn, n, d, Cf, cn, k, lp, lab, md, acc, state, st);
    if (d <= 8) return launch_rowpair<8, 2>(Pf, pn, n, d, Cf, cn, k, lp, lab, md, acc, state, st);
    if (d <= 16) return launch_rowpair<16, 2, 4>(Pf, pn, n, d, Cf, cn, k, lp, lab, md, acc, state, st);
    if (d <= 32) return launch_rowpair<32, 1>(Pf, pn, n, d, Cf, cn, k, lp, lab, md, acc, state, st);
    return PCB_EUNSUP;
  }
  if (variant == PCB_ASSIGN_ROWREG) {
    if (d <= 1) return launch_rowreg<T, 1, 4>(P, pnorm, n, d, C, cnorm, k, lp, lab, mind, acc, state, st);
    if (d <= 2) return launch_rowreg<T, 2, 4>(P, pnorm, n, d, C, cnorm, k, lp, lab, mind, acc, state, st);
    if (d <= 4) return launch_rowreg<T, 4, 4>(P, pnorm, n, d, C, cnorm, k, lp, lab, mind, acc, state, st);
    if (d <= 8) return launch_rowreg<T, 8, 2>(P, pnorm, n, d, C, cnorm, k, lp, lab, mind, acc, state, st);
    if (d <= 16) return launch_rowreg<T, 16, 2>(P, pnorm, n, d, C, cnorm, k, lp, lab, mind, acc, state, st);
    if (d <= 32) return launch_rowreg<T, 32, 1>(P, pnorm, n, d, C, cnorm, k, lp, lab, mind, acc, state, st);
    return PCB_EUNSUP;
  }
  if (variant == PCB_ASSIGN_TILED) {
    auto kern = assign_tiled<T>;
    const int64_t mtiles = (n + TBM - 1) / TBM;
    const int grid = (int)std::min<int64_t>(mtiles, (int64_t)persistent_grid(kern, 256, 0));
    kern<<<grid, 256, 0, st>>>(P, pnorm, n, d, C, cnorm, k, lp, lab, mind, acc, state);
    PCB_CHECK_LAUNCH();
    return 0;
  }
  return PCB_EUNSUP;
}

}  // namespace pcb

extern "C" int pcb_assign_f32(const float* P, const float* pnorm, int64_t n, int d,
                              const float* C, const float* cnorm, int k,
                              const int32_t* labels_prev, int32_t* labels, float* mind,
                              double* acc, const long long* state, int variant, void* stream) {
  if (variant == PCB_ASSIGN_TC3XTF32) return PCB_EUNSUP;  // use pcb_assign_tc_f32
  if (variant == PCB_ASSIGN_DELTA)
    return pcb::assign_delta_f32(P, pnorm, n, d, C, cnorm, k, labels_prev, labels, mind, acc, state,
                                 (cudaStream_t)stream);
  return pcb::assign_dispatch<float>(P, pnorm, n, d, C, cnorm, k, labels_prev, labels, mind, acc,
                                     state, variant, (cudaStream_t)stream);
}

// pcb_assign_f32 whose small-d kernel also applies the changed rows to the
// delta update's sums S when the previous iteration was a delta one (kSpec);
// kernels without the fused path leave that to pcb_delta_update_f32.
extern "C" int pcb_assign_spec_f32(const float* P, const float* pnorm, int64_t n, int d,
                                   const float* C, const float* cnorm, int k,
                                   const int32_t* labels_prev, int32_t* labels, float* mind,
                                   double* acc, const long long* state, double* S, int variant, void* stream) {
  if (variant == PCB_ASSIGN_TC3XTF32 || variant == PCB_ASSIGN_DELTA)
    return pcb_assign_f32(P, pnorm, n, d, C, cnorm, k, labels_prev, labels, mind, acc, state, variant, stream);
  return pcb::assign_dispatch<float>(P, pnorm, n, d, C, cnorm, k, labels_prev, labels, mind, acc, state, variant,
                                     (cudaStream_t)stream, S);
}

extern "C" int pcb_assign_f64(const double* P, const double* pnorm, int64_t n, int d,
                              const double* C, const double* cnorm, int k,
                              const int32_t* labels_prev, int32_t* labels, double* mind,
                              double* acc, const long long* state, int variant, void* stream) {
  if (variant == PCB_ASSIGN_TC3XTF32 || variant == PCB_ASSIGN_DELTA) return PCB_EUNSUP;
  return pcb::assign_dispatch<double>(P, pnorm, n, d, C, cnorm, k, labels_prev, labels, mind, acc,
                                      state, variant, (cudaStream_t)stream);
}
