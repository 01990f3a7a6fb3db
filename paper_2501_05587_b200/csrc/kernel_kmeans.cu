// Kernel K-means (run_popcorn, clustering.py:165-218) on the B200.
//
// The reference builds K = kernel(P P^T) once (kernels.py:85-129: Gram product,
// then an elementwise kernel function), takes point norms from diag(K), and
// per iteration forms E = -2 K V^T with a sparse-dense multiply
// (sparse.py:121-142), z_i = -0.5 E[i, l_i], centroid norms c = V z
// (sparse.py:145-160), D = E + diag(K) + c, then the shared assignment step
// (argmin, empty-cluster repair, objective, changed).
//
// B200 formulation:
//   * Gram + kernel: one tcgen05 3xTF32 GEMM over the upper-triangular 128 x 128
//     tiles of P P^T with the kernel function applied in the epilogue and each
//     tile stored twice (direct + mirrored), so K is exactly symmetric and
//     written once (kernel_gram_tc_kernel); f64 uses a register-tiled SIMT
//     DFMA GEMM with the same epilogue.
//   * E without V: since K is symmetric, (K V^T)[i, j] = (1/|L_j|) sum over
//     m in L_j of K[m, i] - a segmented sum of the ROWS of K in label-sorted
//     order, S[j, :] = sum_{m in L_j} K[m, :] (f64).  That is one coalesced,
//     HBM-bound streaming pass over K per iteration (kk_segsum_kernel), the
//     same counting-sort + segmented-sum machinery as the Lloyd update.
//   * z_i = S[l_i, i] / |L_{l_i}|, c_j = (1/|L_j|) sum_{i in L_j} z_i (f64),
//     D[i, j] = K[i,i] - 2 S[j, i] / |L_j| + c_j (f64), row argmin with the
//     lowest index on ties (kk_assign_kernel) — D is never materialised.
//   * repair (clustering.py:111-139) over the own distances in one block,
//     then counts / objective / changed / history / convergence on the device.
// The per-iteration state machine matches the Lloyd engine (state words,
// stop flag, device-side history), so a whole run enqueues without host sync.
#include <cudaTypedefs.h>

#include "pcb_common.cuh"
#include "pcb_launch.cuh"
#include "screen_common.cuh"
#include "tc_ptx.cuh"

namespace pcb {

// Kernel families (kernels.py:18)
enum KernelFamily { kLinear = 0, kPolynomial = 1, kGaussian = 2, kSigmoid = 3 };

// Elementwise kernel function in the reference's operation order, without
// FMA contraction (numpy evaluates each operator with its own rounding):
//   polynomial: _int_pow(gamma * B + coef, degree)   (kernels.py:96-108, 123)
//   sigmoid:    tanh(gamma * B + coef)
//   gaussian:   exp(max(c * ((-2 B + d_i) + d_j), -88)), c = -gamma / sigma^2
template <typename T>
struct KernelFn {
  int family, degree;
  T gamma, coef, c;
  __device__ __forceinline__ T mul(T a, T b) const;
  __device__ __forceinline__ T add(T a, T b) const;
  __device__ __forceinline__ T apply(T b, T di, T dj) const {
    if (family == kLinear) return b;
    if (family == kGaussian) {
      T e = mul(c, add(add(mul(T(-2), b), di), dj));
      e = e > T(-88) ? e : T(-88);
      return exp(e);
    }
    const T base = add(mul(gamma, b), coef);
    if (family == kSigmoid) return tanh(base);
    // exponentiation by squaring, same multiplication order as _int_pow
    T result = T(0), acc = base;
    bool have = false;
    int e = degree;
    while (e) {
      if (e & 1) {
        result = have ? mul(result, acc) : acc;
        have = true;
      }
      e >>= 1;
      if (e) acc = mul(acc, acc);
    }
    return result;
  }
};
template <> __device__ __forceinline__ float KernelFn<float>::mul(float a, float b) const { return __fmul_rn(a, b); }
template <> __device__ __forceinline__ float KernelFn<float>::add(float a, float b) const { return __fadd_rn(a, b); }
template <> __device__ __forceinline__ double KernelFn<double>::mul(double a, double b) const { return __dmul_rn(a, b); }
template <> __device__ __forceinline__ double KernelFn<double>::add(double a, double b) const { return __dadd_rn(a, b); }

// upper-triangular tile index t -> (I, J), I <= J, row-major over I
__device__ __forceinline__ void upper_tile(int64_t t, int nt, int& I, int& J) {
  // rows 0..I-1 hold I*nt - I(I-1)/2 tiles
  double a = 2.0 * nt + 1.0;
  int i = (int)floor((a - sqrt(a * a - 8.0 * (double)t)) * 0.5);
  if (i < 0) i = 0;
  if (i > nt - 1) i = nt - 1;
  auto start = [nt](int r) { return (int64_t)r * nt - (int64_t)r * (r - 1) / 2; };
  while (i > 0 && start(i) > t) --i;
  while (i + 1 < nt && start(i + 1) <= t) ++i;
  I = i;
  J = i + (int)(t - start(i));
}

// ---------------------------------------------------------------------------
// Gram + kernel, f32: tcgen05 3xTF32, 128 x 128 upper tiles, mirrored stores
// ---------------------------------------------------------------------------
constexpr int GT_B = 128;       // tile edge (UMMA M = N = 128)
constexpr int GT_BK = 32;
constexpr int GT_STAGES = 3;
constexpr int GT_THREADS = 384;  // 4 control warps + 8 epilogue warps (2 per TMEM lane group)
constexpr uint32_t GT_TILE_BYTES = GT_B * GT_BK * 4;                 // 16 KB
constexpr uint32_t GT_STAGE_BYTES = 4 * GT_TILE_BYTES;               // A hi/lo, B hi/lo
constexpr uint32_t GT_SMEM = 1024 + GT_STAGES * GT_STAGE_BYTES + 1024 + 8 * 32 * 33 * 4;

__global__ void __launch_bounds__(GT_THREADS, 1)
kernel_gram_tc_kernel(const __grid_constant__ CUtensorMap tm_hi, const __grid_constant__ CUtensorMap tm_lo,
                      const __grid_constant__ CUtensorMap tm_bhi, const __grid_constant__ CUtensorMap tm_blo,
                      int64_t n, int64_t nb, bool sym, int num_kc, const float* __restrict__ dvec,
                      const float* __restrict__ dvec_b, float* __restrict__ K, int64_t ldk, KernelFn<float> fn,
                      unsigned long long* __restrict__ nonfinite) {
  // sym: K = kernel(A A^T) over the upper tiles, mirrored (B maps unused);
  // else K (n x nb) = kernel(A B^T) over all tiles (kernel_matrix_between).
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw & 1023u)) & 1023u);
  uint8_t* bar_area = smem + GT_STAGES * GT_STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(bar_area);
  uint64_t* empty = full + GT_STAGES;
  uint64_t* tfull = empty + GT_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tm_hi);
    ptx::prefetch_tmap(&tm_lo);
    if (!sym) {
      ptx::prefetch_tmap(&tm_bhi);
      ptx::prefetch_tmap(&tm_blo);
    }
    for (int s = 0; s < GT_STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], 256);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<256>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int nt = (int)((n + GT_B - 1) / GT_B);
  const int ntb = (int)((nb + GT_B - 1) / GT_B);
  const int64_t ntiles = sym ? (int64_t)nt * (nt + 1) / 2 : (int64_t)nt * ntb;
  auto tile_of = [&](int64_t t, int& I, int& J) {
    if (sym) {
      upper_tile(t, nt, I, J);
    } else {
      I = (int)(t / ntb);
      J = (int)(t % ntb);
    }
  };
  const CUtensorMap* bhi = sym ? &tm_hi : &tm_bhi;
  const CUtensorMap* blo = sym ? &tm_lo : &tm_blo;

  if (warp == 0) {
    int stage = 0;
    uint32_t phase = 0;
    const uint64_t pol = ptx::policy_evict_last();
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int I, J;
      tile_of(t, I, J);
      for (int kc = 0; kc < num_kc; ++kc) {
        ptx::mbar_wait(&empty[stage], phase ^ 1u);
        uint8_t* st = smem + stage * GT_STAGE_BYTES;
        if (ptx::elect_one()) {
          ptx::mbar_expect_tx(&full[stage], GT_STAGE_BYTES);
          ptx::tma_load_2d(&tm_hi, &full[stage], st, kc * GT_BK, I * GT_B, pol);
          ptx::tma_load_2d(&tm_lo, &full[stage], st + GT_TILE_BYTES, kc * GT_BK, I * GT_B, pol);
          ptx::tma_load_2d(bhi, &full[stage], st + 2 * GT_TILE_BYTES, kc * GT_BK, J * GT_B, pol);
          ptx::tma_load_2d(blo, &full[stage], st + 3 * GT_TILE_BYTES, kc * GT_BK, J * GT_B, pol);
        }
        __syncwarp();
        if (++stage == GT_STAGES) { stage = 0; phase ^= 1u; }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = ptx::idesc_tf32<GT_B, GT_B>();
    int stage = 0;
    uint32_t phase = 0;
    int abuf = 0;
    uint32_t aphase = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      ptx::mbar_wait(&tempty[abuf], aphase ^ 1u);
      ptx::tc_fence_after();
      const uint32_t dt = tmem + (uint32_t)(abuf * GT_B);
      for (int kc = 0; kc < num_kc; ++kc) {
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        const uint32_t base = ptx::smem_u32(smem + stage * GT_STAGE_BYTES);
        const uint64_t ahi = ptx::sdesc_k_sw128(base);
        const uint64_t alo = ptx::sdesc_k_sw128(base + GT_TILE_BYTES);
        const uint64_t bhi = ptx::sdesc_k_sw128(base + 2 * GT_TILE_BYTES);
        const uint64_t blo = ptx::sdesc_k_sw128(base + 3 * GT_TILE_BYTES);
        if (ptx::elect_one()) {
#pragma unroll
          for (int ks = 0; ks < GT_BK / 8; ++ks) {
            const uint64_t off = (uint64_t)(ks * 8 * 4) >> 4;
            ptx::umma_tf32(dt, ahi + off, bhi + off, idesc, (kc | ks) != 0);
            ptx::umma_tf32(dt, ahi + off, blo + off, idesc, 1u);
            ptx::umma_tf32(dt, alo + off, bhi + off, idesc, 1u);
          }
          ptx::umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == GT_STAGES) { stage = 0; phase ^= 1u; }
      }
      if (ptx::elect_one()) ptx::umma_commit(&tfull[abuf]);
      __syncwarp();
      abuf ^= 1;
      if (abuf == 0) aphase ^= 1u;
    }
  } else if (warp >= 4) {
    // warp (ew, h): TMEM lane group ew = warp % 4, column half h (64 columns)
    const int ew = warp & 3, h = (warp - 4) >> 2;
    float* xt = reinterpret_cast<float*>(bar_area + 1024) + (warp - 4) * 32 * 33;  // per-warp transpose tile
    int abuf = 0;
    uint32_t aphase = 0;
    bool bad = false;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int I, J;
      tile_of(t, I, J);
      const int64_t row = (int64_t)I * GT_B + ew * 32 + lane;
      const int64_t ncol = sym ? n : nb;
      const float* dv_col = sym ? dvec : dvec_b;
      const float di = (fn.family == kGaussian && row < n) ? dvec[row] : 0.0f;
      ptx::mbar_wait(&tfull[abuf], aphase);
      ptx::tc_fence_after();
      const uint32_t taddr = tmem + ((uint32_t)(ew * 32) << 16) + (uint32_t)(abuf * GT_B);
#pragma unroll 1
      for (int cb = h * 64; cb < h * 64 + 64; cb += 32) {
        float v[32];
        ptx::tmem_ld_32x32b_x32(taddr + cb, v);
        const int64_t c0 = (int64_t)J * GT_B + cb;
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const int64_t col = c0 + c;
          const float dj = (fn.family == kGaussian && col < ncol) ? __ldg(&dv_col[col]) : 0.0f;
          float x = fn.apply(v[c], di, dj);
          if (sym && fn.family == kGaussian && col == row) x = 1.0f;  // fill_diagonal(K, 1.0)
          v[c] = x;
        }
        // direct stores: row `row`, columns c0.. (upper part only on diagonal
        // tiles), transposed through shared memory so that every warp store
        // writes 32 consecutive floats of one row (thread = column)
        {
          const int64_t row0 = (int64_t)I * GT_B + ew * 32;
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const int64_t col = c0 + c;
            if (row < n && col < ncol && (!sym || I != J || col >= row)) bad |= !isfinite(v[c]);
            xt[lane * 33 + c] = v[c];
          }
          __syncwarp();
          const int64_t col = c0 + lane;
#pragma unroll 4
          for (int r = 0; r < 32; ++r) {
            const int64_t rr = row0 + r;
            if (rr < n && col < ncol && (!sym || I != J || col >= rr)) K[rr * ldk + col] = xt[r * 33 + lane];
          }
          __syncwarp();
        }
        // mirrored stores: column `row` of rows c0.. (a warp writes 32 consecutive floats per c)
        if (sym)
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const int64_t col = c0 + c;
          if (row < n && col < n && (I != J ? true : col > row)) K[col * ldk + row] = v[c];
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[abuf]);
      abuf ^= 1;
      if (abuf == 0) aphase ^= 1u;
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicAdd(nonfinite, 1ull);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc<256>(tmem);
}

// ---------------------------------------------------------------------------
// Gram + kernel, f64 (and small fallback): register-tiled SIMT, 64 x 64 tiles
// ---------------------------------------------------------------------------
constexpr int GS_B = 64;
constexpr int GS_BK = 16;

template <typename T>
__global__ void __launch_bounds__(256)
kernel_gram_simt_kernel(const T* __restrict__ P, int64_t n, const T* __restrict__ Q, int64_t nq, bool sym, int d,
                        const T* __restrict__ dvec, const T* __restrict__ dvec_q, T* __restrict__ K, int64_t ldk,
                        KernelFn<T> fn, unsigned long long* __restrict__ nonfinite) {
  // sym: K = kernel(P P^T) (upper tiles, mirrored); else K (n x nq) = kernel(P Q^T)
  __shared__ T As[GS_BK][GS_B + 1];
  __shared__ T Bs[GS_BK][GS_B + 1];
  const int nt = (int)((n + GS_B - 1) / GS_B);
  const int ntq = (int)((nq + GS_B - 1) / GS_B);
  const int64_t ntiles = sym ? (int64_t)nt * (nt + 1) / 2 : (int64_t)nt * ntq;
  const T* Qs = sym ? P : Q;
  const T* dq = sym ? dvec : dvec_q;
  const int64_t ncol = sym ? n : nq;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, 4 x 4 outputs each
  bool bad = false;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int I, J;
    if (sym) {
      upper_tile(t, nt, I, J);
    } else {
      I = (int)(t / ntq);
      J = (int)(t % ntq);
    }
    const int64_t r0 = (int64_t)I * GS_B, c0 = (int64_t)J * GS_B;
    T acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = T(0);
    for (int k0 = 0; k0 < d; k0 += GS_BK) {
      __syncthreads();
      for (int e = threadIdx.x; e < GS_BK * GS_B; e += blockDim.x) {
        const int kk = e % GS_BK, r = e / GS_BK;
        const int64_t gr = r0 + r, gc = c0 + r;
        As[kk][r] = (gr < n && k0 + kk < d) ? P[gr * d + k0 + kk] : T(0);
        Bs[kk][r] = (gc < ncol && k0 + kk < d) ? Qs[gc * d + k0 + kk] : T(0);
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < GS_BK; ++kk) {
        T a[4], b[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          a[q] = As[kk][ty + 16 * q];
          b[q] = Bs[kk][tx + 16 * q];
        }
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[p][q] = fma(a[p], b[q], acc[p][q]);
      }
    }
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int64_t row = r0 + ty + 16 * p;
      if (row >= n) continue;
      const T di = fn.family == kGaussian ? dvec[row] : T(0);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t col = c0 + tx + 16 * q;
        if (col >= ncol || (sym && I == J && col < row)) continue;
        const T dj = fn.family == kGaussian ? dq[col] : T(0);
        T x = fn.apply(acc[p][q], di, dj);
        if (sym && fn.family == kGaussian && col == row) x = T(1);
        K[row * ldk + col] = x;
        if (sym && col != row) K[col * ldk + row] = x;
        bad |= !isfinite(x);
      }
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicAdd(nonfinite, 1ull);
}

// ---------------------------------------------------------------------------
// per-iteration kernels
// ---------------------------------------------------------------------------
// Kernel-path accumulator (f64, zeroed per iteration):
//   [ counts of the new labels k | cnsum k | objective | changed ]
struct KkLayout {
  int64_t k;
  __host__ __device__ int64_t counts() const { return 0; }
  __host__ __device__ int64_t cnsum() const { return k; }
  __host__ __device__ int64_t objective() const { return 2 * k; }
  __host__ __device__ int64_t changed() const { return 2 * k + 1; }
};

// S[j, c] += sum over sorted positions s in segment j of K[perm[s], c]
// grid: x = column tiles of 4 * blockDim.x, y = chunks of sorted positions
template <typename T, int VEC>
__global__ void __launch_bounds__(256)
kk_segsum_kernel(const T* __restrict__ K, int64_t ldk, int64_t n, int64_t ncols,
                 const int32_t* __restrict__ perm, const int32_t* __restrict__ offsets, int k,
                 double* __restrict__ S, int64_t lds, int64_t chunk, const long long* __restrict__ state) {
  if (stopped(state)) return;
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * VEC;
  const int64_t s0 = (int64_t)blockIdx.y * chunk;
  const int64_t s1 = min(n, s0 + chunk);
  if (s0 >= s1) return;
  // segment containing s0: last j with offsets[j] <= s0
  int lo = 0, hi = k;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (offsets[mid] <= s0) lo = mid;
    else hi = mid - 1;
  }
  int seg = lo;
  int64_t seg_end = offsets[seg + 1];
  double acc[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) acc[v] = 0.0;
  bool dirty = false;
  const bool in = c < ncols;
  auto flush = [&]() {
    if (dirty && in) {
#pragma unroll
      for (int v = 0; v < VEC; ++v)
        if (c + v < ncols) atomicAdd(&S[(int64_t)seg * lds + c + v], acc[v]);
    }
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[v] = 0.0;
    dirty = false;
  };
  // software pipeline: K rows of batch i+1 are in flight while batch i is
  // accumulated, and their perm[] entries were fetched one batch earlier.
  // K is streamed once per iteration (>> L2): loads are evict-first (.cs).
  constexpr int U = 4;
  auto load_perm = [&](int64_t sb, int (&p)[U]) {
#pragma unroll
    for (int u = 0; u < U; ++u) p[u] = (sb + u < s1) ? __ldg(&perm[sb + u]) : -1;
  };
  auto load_x = [&](const int (&p)[U], T (&x)[U][VEC]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (p[u] >= 0 && in) {
        const T* src = K + (int64_t)p[u] * ldk + c;
        if constexpr (VEC == 4) {
          const float4 q = __ldcs(reinterpret_cast<const float4*>(src));
          x[u][0] = q.x; x[u][1] = q.y; x[u][2] = q.z; x[u][3] = q.w;
        } else {
          const double2 q = __ldcs(reinterpret_cast<const double2*>(src));
          x[u][0] = q.x; x[u][1] = q.y;
        }
      } else {
#pragma unroll
        for (int v = 0; v < VEC; ++v) x[u][v] = T(0);
      }
    }
  };
  auto accum = [&](int64_t sb, const T (&x)[U][VEC]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (sb + u >= s1) break;
      while (sb + u >= seg_end) {  // next non-empty segment
        flush();
        ++seg;
        seg_end = offsets[seg + 1];
      }
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[v] += (double)x[u][v];
      dirty = true;
    }
  };
  int pa[U], pb[U];
  T xa[U][VEC], xb[U][VEC];
  load_perm(s0, pa);
  load_x(pa, xa);
  load_perm(s0 + U, pb);
  for (int64_t s = s0; s < s1; s += 2 * U) {
    load_x(pb, xb);            // rows of batch s + U
    load_perm(s + 2 * U, pa);  // perm of batch s + 2U
    accum(s, xa);
    load_x(pa, xa);            // rows of batch s + 2U
    load_perm(s + 3 * U, pb);
    accum(s + U, xb);
  }
  flush();
}

// cnsum[l_i] += S[l_i, i] / |L_{l_i}|   (z of sparse.py's spmv, clustering.py:199-200)
__global__ void kk_centroid_terms_kernel(const double* __restrict__ S, int64_t lds, int64_t n,
                                         const double* __restrict__ cnt, const int32_t* __restrict__ labels,
                                         double* __restrict__ acc, int k, const long long* __restrict__ state) {
  if (stopped(state)) return;
  const KkLayout L{k};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int l = labels[i];
    atomicAdd(&acc[L.cnsum() + l], S[(int64_t)l * lds + i] / cnt[l]);
  }
}

// D[i, j] = K[i,i] - 2 S[j,i] / |L_j| + cnsum_j / |L_j|, argmin (lowest j on
// ties), own distance, int counts of the raw labels (for repair).
template <typename T>
__global__ void __launch_bounds__(256)
kk_assign_kernel(const T* __restrict__ K, int64_t ldk, const double* __restrict__ S, int64_t lds, int64_t n,
                 int k, const double* __restrict__ cnt, const double* __restrict__ acc,
                 int32_t* __restrict__ labels, double* __restrict__ own, int* __restrict__ icounts,
                 long long* __restrict__ state) {
  if (stopped(state)) return;
  extern __shared__ double sh[];  // [k] 2/|L_j|, [k] c_j
  const KkLayout L{k};
  double* two_inv = sh;
  double* cterm = sh + k;
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    const double inv = 1.0 / cnt[j];
    two_inv[j] = 2.0 * inv;
    cterm[j] = acc[L.cnsum() + j] * inv;
  }
  __syncthreads();
  bool nan_seen = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double pn = (double)K[i * ldk + i];
    double best = INFINITY;
    int bj = 0;
    for (int j = 0; j < k; ++j) {
      const double dij = (pn - two_inv[j] * S[(int64_t)j * lds + i]) + cterm[j];
      nan_seen |= isnan(dij);
      if (dij < best) { best = dij; bj = j; }
    }
    labels[i] = bj;
    own[i] = best;
    atomicAdd(&icounts[bj], 1);
  }
  if (__syncthreads_or(nan_seen) && threadIdx.x == 0) atomicExch((unsigned long long*)&state[kNanFlag], 1ull);
}

// Empty-cluster repair (clustering.py:111-139) in one block: while a cluster
// is empty, for each empty j ascending move the unmoved point with the
// largest own distance (lowest index on ties) to j.  moved[] marks donors.
template <typename T>
__global__ void __launch_bounds__(1024)
kk_repair_kernel(const T* __restrict__ K, int64_t ldk, const double* __restrict__ S, int64_t lds, int64_t n,
                 int k, const double* __restrict__ cnt, const double* __restrict__ acc,
                 int32_t* __restrict__ labels, double* __restrict__ own, int* __restrict__ icounts,
                 uint8_t* __restrict__ moved, int* __restrict__ elist, long long* __restrict__ state) {
  if (stopped(state)) return;
  __shared__ int s_any;
  __shared__ double s_v[32];
  __shared__ long long s_i[32];
  if (threadIdx.x == 0) s_any = 0;
  __syncthreads();
  for (int j = threadIdx.x; j < k; j += blockDim.x)
    if (icounts[j] == 0) s_any = 1;
  __syncthreads();
  if (!s_any) return;
  const KkLayout L{k};
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) moved[i] = 0;
  long long nmoved = 0;
  while (true) {
    __syncthreads();
    if (threadIdx.x == 0) {
      int c = 0;
      for (int j = 0; j < k; ++j)
        if (icounts[j] == 0) elist[1 + c++] = j;
      elist[0] = c;
    }
    __syncthreads();
    const int ne = elist[0];
    if (ne == 0) break;
    for (int e = 0; e < ne; ++e) {
      const int j = elist[1 + e];
      double bv = -INFINITY;
      long long bi = n;
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double v = moved[i] ? -INFINITY : own[i];
        if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
        const long long i2 = __shfl_xor_sync(0xffffffffu, bi, o);
        if (v2 > bv || (v2 == bv && i2 < bi)) { bv = v2; bi = i2; }
      }
      if ((threadIdx.x & 31) == 0) { s_v[threadIdx.x >> 5] = bv; s_i[threadIdx.x >> 5] = bi; }
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
          if (s_v[w] > bv || (s_v[w] == bv && s_i[w] < bi)) { bv = s_v[w]; bi = s_i[w]; }
        const int64_t donor = bi < n ? bi : 0;  // k <= n guarantees an unmoved donor
        const int old = labels[donor];
        labels[donor] = j;
        moved[donor] = 1;
        icounts[old] -= 1;
        icounts[j] += 1;
        // the donor's entry of the (fixed) distance matrix of this iteration
        const double inv = 1.0 / cnt[j];
        own[donor] = ((double)K[donor * ldk + donor] - 2.0 * inv * S[(int64_t)j * lds + donor]) +
                     acc[L.cnsum() + j] * inv;
        ++nmoved;
      }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) state[kMoved] += nmoved;
}

// counts (f64) of the final labels, objective = sum own, changed
__global__ void kk_bookkeep_kernel(const int32_t* __restrict__ labels, const int32_t* __restrict__ prev,
                                   const double* __restrict__ own, int64_t n, int k, double* __restrict__ acc,
                                   const long long* __restrict__ state) {
  if (stopped(state)) return;
  extern __shared__ int hist[];
  const KkLayout L{k};
  for (int j = threadIdx.x; j < k; j += blockDim.x) hist[j] = 0;
  __syncthreads();
  double obj = 0.0;
  long long chg = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int l = labels[i];
    atomicAdd(&hist[l], 1);
    obj += own[i];
    if (prev) chg += (prev[i] != l);
  }
  obj = warp_sum(obj);
  chg = warp_sum(chg);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&acc[L.objective()], obj);
    if (chg) atomicAdd(&acc[L.changed()], (double)chg);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < k; j += blockDim.x)
    if (hist[j]) atomicAdd(&acc[L.counts() + j], (double)hist[j]);
}

// history + convergence (clustering.py:204-216); counts of the new labels become current
__global__ void kk_finalize_kernel(const double* __restrict__ acc, int k, int64_t n_total,
                                   double* __restrict__ cnt, double* __restrict__ obj_hist,
                                   long long* __restrict__ rep_hist, long long* __restrict__ state,
                                   int check_convergence, double tol) {
  if (stopped(state)) return;
  const KkLayout L{k};
  for (int j = threadIdx.x; j < k; j += blockDim.x) cnt[j] = acc[L.counts() + j];
  if (threadIdx.x != 0) return;
  const long long it = state[kIters];
  obj_hist[it] = acc[L.objective()];
  rep_hist[it] = state[kMoved];
  state[kMoved] = 0;
  state[kIters] = it + 1;
  if (check_convergence && acc[L.changed()] / (double)n_total <= tol) {
    state[kConverged] = 1;
    state[kStop] = 1;
  }
}

static int make_tmap_rows_f32(CUtensorMap* m, const float* base, int64_t rows, int cols) {
  return make_tmap_rows(m, base, rows, cols, GT_B);
}

template <typename T>
static KernelFn<T> make_fn(int family, double gamma, double coef, int degree, double sigma) {
  KernelFn<T> f;
  f.family = family;
  f.degree = degree;
  f.gamma = (T)gamma;
  f.coef = (T)coef;
  f.c = (T)(-gamma / (sigma * sigma));
  return f;
}

}  // namespace pcb

using namespace pcb;

static bool bad_family(int family, int degree, double sigma) {
  if (family < kLinear || family > kSigmoid) return true;
  if ((family == kPolynomial) && degree < 1) return true;
  if (family == kGaussian && !(sigma > 0)) return true;
  return false;
}

extern "C" int pcb_kernel_gram_f32(const float* P_hi, const float* P_lo, int ld, int64_t n, const float* dvec,
                                   float* K, int64_t ldk, int family, double gamma, double coef, int degree,
                                   double sigma, unsigned long long* nonfinite, void* stream) {
  if (n < 1 || ld < 1 || ld % GT_BK != 0 || ldk < n || !P_hi || !P_lo || !K || !nonfinite) return PCB_EINVAL;
  if (bad_family(family, degree, sigma) || (family == kGaussian && !dvec)) return PCB_EINVAL;
  if (n > INT32_MAX) return PCB_EUNSUP;
  CUtensorMap thi, tlo;
  int rc;
  if ((rc = make_tmap_rows_f32(&thi, P_hi, n, ld))) return rc;
  if ((rc = make_tmap_rows_f32(&tlo, P_lo, n, ld))) return rc;
  cudaError_t e = cudaFuncSetAttribute(kernel_gram_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)GT_SMEM);
  if (e != cudaSuccess) return (int)e;
  const int64_t nt = (n + GT_B - 1) / GT_B;
  const int grid = (int)std::min<int64_t>(nt * (nt + 1) / 2, (int64_t)sm_count());
  kernel_gram_tc_kernel<<<grid, GT_THREADS, GT_SMEM, (cudaStream_t)stream>>>(
      thi, tlo, thi, tlo, n, n, true, ld / GT_BK, dvec, dvec, K, ldk,
      make_fn<float>(family, gamma, coef, degree, sigma), nonfinite);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_kernel_cross_f32(const float* A_hi, const float* A_lo, int64_t na, const float* B_hi,
                                    const float* B_lo, int64_t nb, int ld, const float* dva, const float* dvb,
                                    float* K, int64_t ldk, int family, double gamma, double coef, int degree,
                                    double sigma, unsigned long long* nonfinite, void* stream) {
  if (na < 1 || nb < 1 || ld < 1 || ld % GT_BK != 0 || ldk < nb || !A_hi || !A_lo || !B_hi || !B_lo || !K ||
      !nonfinite)
    return PCB_EINVAL;
  if (bad_family(family, degree, sigma) || (family == kGaussian && (!dva || !dvb))) return PCB_EINVAL;
  if (na > INT32_MAX || nb > INT32_MAX) return PCB_EUNSUP;
  CUtensorMap ahi, alo, bhi, blo;
  int rc;
  if ((rc = make_tmap_rows_f32(&ahi, A_hi, na, ld))) return rc;
  if ((rc = make_tmap_rows_f32(&alo, A_lo, na, ld))) return rc;
  if ((rc = make_tmap_rows_f32(&bhi, B_hi, nb, ld))) return rc;
  if ((rc = make_tmap_rows_f32(&blo, B_lo, nb, ld))) return rc;
  cudaError_t e = cudaFuncSetAttribute(kernel_gram_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)GT_SMEM);
  if (e != cudaSuccess) return (int)e;
  const int64_t tiles = ((na + GT_B - 1) / GT_B) * ((nb + GT_B - 1) / GT_B);
  const int grid = (int)std::min<int64_t>(tiles, (int64_t)sm_count());
  kernel_gram_tc_kernel<<<grid, GT_THREADS, GT_SMEM, (cudaStream_t)stream>>>(
      ahi, alo, bhi, blo, na, nb, false, ld / GT_BK, dva, dvb, K, ldk,
      make_fn<float>(family, gamma, coef, degree, sigma), nonfinite);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_kernel_gram_f64(const double* P, int64_t n, int d, const double* dvec, double* K, int64_t ldk,
                                   int family, double gamma, double coef, int degree, double sigma,
                                   unsigned long long* nonfinite, void* stream) {
  if (n < 1 || d < 1 || ldk < n || !P || !K || !nonfinite) return PCB_EINVAL;
  if (bad_family(family, degree, sigma) || (family == kGaussian && !dvec)) return PCB_EINVAL;
  const int64_t nt = (n + GS_B - 1) / GS_B;
  const int grid = (int)std::min<int64_t>(nt * (nt + 1) / 2, (int64_t)sm_count() * 4);
  kernel_gram_simt_kernel<double><<<grid, 256, 0, (cudaStream_t)stream>>>(
      P, n, P, n, true, d, dvec, dvec, K, ldk, make_fn<double>(family, gamma, coef, degree, sigma), nonfinite);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_kernel_cross_f64(const double* A, int64_t na, const double* B, int64_t nb, int d,
                                    const double* dva, const double* dvb, double* K, int64_t ldk, int family,
                                    double gamma, double coef, int degree, double sigma,
                                    unsigned long long* nonfinite, void* stream) {
  if (na < 1 || nb < 1 || d < 1 || ldk < nb || !A || !B || !K || !nonfinite) return PCB_EINVAL;
  if (bad_family(family, degree, sigma) || (family == kGaussian && (!dva || !dvb))) return PCB_EINVAL;
  const int64_t tiles = ((na + GS_B - 1) / GS_B) * ((nb + GS_B - 1) / GS_B);
  const int grid = (int)std::min<int64_t>(tiles, (int64_t)sm_count() * 4);
  kernel_gram_simt_kernel<double><<<grid, 256, 0, (cudaStream_t)stream>>>(
      A, na, B, nb, false, d, dva, dvb, K, ldk, make_fn<double>(family, gamma, coef, degree, sigma), nonfinite);
  PCB_CHECK_LAUNCH();
  return 0;
}

template <typename T>
static int kk_segment_sums(const T* K, int64_t ldk, int64_t n, int64_t ncols, const int32_t* perm,
                           const int32_t* offsets, int k, double* S, int64_t lds, const long long* state,
                           cudaStream_t st) {
  if (n < 1 || ncols < 1 || k < 1 || ldk < ncols || lds < ncols || !K || !perm || !offsets || !S)
    return PCB_EINVAL;
  constexpr int VEC = sizeof(T) == 4 ? 4 : 2;
  if (ldk % VEC != 0) return PCB_EINVAL;
  cudaError_t e = cudaMemsetAsync(S, 0, sizeof(double) * (size_t)k * (size_t)lds, st);
  if (e != cudaSuccess) return (int)e;
  const int64_t colblocks = (ncols + 256 * VEC - 1) / (256 * VEC);
  // many small work items (~32 per SM) so the hardware scheduler balances the
  // SMs; each chunk at least 128 rows (one flush per segment boundary)
  int64_t chunks = std::max<int64_t>(1, (32 * (int64_t)sm_count() + colblocks - 1) / colblocks);
  chunks = std::min<int64_t>(chunks, std::max<int64_t>(1, n / 128));
  chunks = std::min<int64_t>(chunks, 65535);
  const int64_t chunk = (n + chunks - 1) / chunks;
  dim3 grid((unsigned)colblocks, (unsigned)chunks);
  kk_segsum_kernel<T, VEC><<<grid, 256, 0, st>>>(K, ldk, n, ncols, perm, offsets, k, S, lds, chunk, state);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_kk_segment_sums_f32(const float* K, int64_t ldk, int64_t n, int64_t ncols,
                                       const int32_t* perm, const int32_t* offsets, int k, double* S, int64_t lds,
                                       const long long* state, void* stream) {
  return kk_segment_sums<float>(K, ldk, n, ncols, perm, offsets, k, S, lds, state, (cudaStream_t)stream);
}

extern "C" int pcb_kk_segment_sums_f64(const double* K, int64_t ldk, int64_t n, int64_t ncols,
                                       const int32_t* perm, const int32_t* offsets, int k, double* S, int64_t lds,
                                       const long long* state, void* stream) {
  return kk_segment_sums<double>(K, ldk, n, ncols, perm, offsets, k, S, lds, state, (cudaStream_t)stream);
}

// ---- predict (estimator.py:131-147, kernel drivers) ------------------------
// D[i, j] = self_i - 2 S[j, i] / |L_j| + cself_j, self_i = _self_kernel(x_i)
// (estimator.py:163-171) from xn = |x_i|^2; argmin, lowest j on ties.
template <typename T>
__global__ void kk_predict_kernel(const double* __restrict__ S, int64_t lds, int64_t m, int k,
                                  const double* __restrict__ cnt, const double* __restrict__ cself,
                                  const T* __restrict__ xn, KernelFn<T> fn, int32_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const T sq = xn[i];
    T self;
    if (fn.family == kLinear) self = sq;
    else if (fn.family == kGaussian) self = T(1);
    else if (fn.family == kSigmoid) self = tanh(fn.add(fn.mul(fn.gamma, sq), fn.coef));
    else self = pow(fn.add(fn.mul(fn.gamma, sq), fn.coef), (T)fn.degree);
    double best = INFINITY;
    int bj = 0;
    for (int j = 0; j < k; ++j) {
      const double mj = cnt[j] > 0 ? cnt[j] : 1.0;
      const double dij = ((double)self - (2.0 / mj) * S[(int64_t)j * lds + i]) + cself[j];
      if (dij < best) { best = dij; bj = j; }
    }
    out[i] = bj;
  }
}

extern "C" int pcb_kk_predict_f32(const double* S, int64_t lds, int64_t m, int k, const double* cnt,
                                  const double* cself, const float* xn, int family, double gamma, double coef,
                                  int degree, double sigma, int32_t* out, void* stream) {
  if (m < 1 || k < 1 || !S || !cnt || !cself || !xn || !out || bad_family(family, degree, sigma)) return PCB_EINVAL;
  const int g = (int)std::min<int64_t>((m + 255) / 256, 8L * sm_count());
  kk_predict_kernel<float><<<g, 256, 0, (cudaStream_t)stream>>>(S, lds, m, k, cnt, cself, xn,
                                                                 make_fn<float>(family, gamma, coef, degree, sigma), out);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_kk_predict_f64(const double* S, int64_t lds, int64_t m, int k, const double* cnt,
                                  const double* cself, const double* xn, int family, double gamma, double coef,
                                  int degree, double sigma, int32_t* out, void* stream) {
  if (m < 1 || k < 1 || !S || !cnt || !cself || !xn || !out || bad_family(family, degree, sigma)) return PCB_EINVAL;
  const int g = (int)std::min<int64_t>((m + 255) / 256, 8L * sm_count());
  kk_predict_kernel<double><<<g, 256, 0, (cudaStream_t)stream>>>(S, lds, m, k, cnt, cself, xn,
                                                                   make_fn<double>(family, gamma, coef, degree, sigma),
                                                                   out);
  PCB_CHECK_LAUNCH();
  return 0;
}

template <typename T>
static int kk_assign(const T* K, int64_t ldk, const double* S, int64_t lds, int64_t n, int k, const double* cnt,
                     double* acc, const int32_t* labels_cur, int32_t* labels_new, double* own, int* icounts,
                     long long* state, cudaStream_t st) {
  if (n < 1 || k < 1 || !K || !S || !cnt || !acc || !labels_cur || !labels_new || !own || !icounts || !state)
    return PCB_EINVAL;
  if ((size_t)k * 16 > 200 * 1024) return PCB_EUNSUP;
  cudaError_t e = cudaMemsetAsync(icounts, 0, sizeof(int) * (size_t)k, st);
  if (e != cudaSuccess) return (int)e;
  const int g = (int)std::min<int64_t>((n + 255) / 256, 8L * sm_count());
  kk_centroid_terms_kernel<<<g, 256, 0, st>>>(S, lds, n, cnt, labels_cur, acc, k, state);
  PCB_CHECK_LAUNCH();
  const size_t sm = (size_t)k * 16;
  if (sm > 48 * 1024) {
    e = cudaFuncSetAttribute(kk_assign_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return (int)e;
  }
  kk_assign_kernel<T><<<g, 256, sm, st>>>(K, ldk, S, lds, n, k, cnt, acc, labels_new, own, icounts, state);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_kk_assign_f32(const float* K, int64_t ldk, const double* S, int64_t lds, int64_t n, int k,
                                 const double* cnt, double* acc, const int32_t* labels_cur, int32_t* labels_new,
                                 double* own, int* icounts, long long* state, void* stream) {
  return kk_assign<float>(K, ldk, S, lds, n, k, cnt, acc, labels_cur, labels_new, own, icounts, state,
                          (cudaStream_t)stream);
}

extern "C" int pcb_kk_assign_f64(const double* K, int64_t ldk, const double* S, int64_t lds, int64_t n, int k,
                                 const double* cnt, double* acc, const int32_t* labels_cur, int32_t* labels_new,
                                 double* own, int* icounts, long long* state, void* stream) {
  return kk_assign<double>(K, ldk, S, lds, n, k, cnt, acc, labels_cur, labels_new, own, icounts, state,
                           (cudaStream_t)stream);
}

extern "C" int64_t pcb_kk_repair_scratch_bytes(int64_t n, int k) {
  if (n < 1 || k < 1) return PCB_EINVAL;
  return (int64_t)(((size_t)n + 255) / 256 * 256 + sizeof(int) * ((size_t)k + 1));
}

template <typename T>
static int kk_repair(const T* K, int64_t ldk, const double* S, int64_t lds, int64_t n, int k, const double* cnt,
                     const double* acc, int32_t* labels, double* own, int* icounts, long long* state,
                     void* scratch, int64_t bytes, cudaStream_t st) {
  if (n < 1 || k < 1 || !K || !S || !cnt || !acc || !labels || !own || !icounts || !state || !scratch)
    return PCB_EINVAL;
  if (bytes < pcb_kk_repair_scratch_bytes(n, k)) return PCB_EINVAL;
  uint8_t* moved = (uint8_t*)scratch;
  int* elist = (int*)((uint8_t*)scratch + ((size_t)n + 255) / 256 * 256);
  kk_repair_kernel<T><<<1, 1024, 0, st>>>(K, ldk, S, lds, n, k, cnt, acc, labels, own, icounts, moved, elist,
                                          state);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_kk_repair_f32(const float* K, int64_t ldk, const double* S, int64_t lds, int64_t n, int k,
                                 const double* cnt, const double* acc, int32_t* labels, double* own, int* icounts,
                                 long long* state, void* scratch, int64_t bytes, void* stream) {
  return kk_repair<float>(K, ldk, S, lds, n, k, cnt, acc, labels, own, icounts, state, scratch, bytes,
                          (cudaStream_t)stream);
}

extern "C" int pcb_kk_repair_f64(const double* K, int64_t ldk, const double* S, int64_t lds, int64_t n, int k,
                                 const double* cnt, const double* acc, int32_t* labels, double* own, int* icounts,
                                 long long* state, void* scratch, int64_t bytes, void* stream) {
  return kk_repair<double>(K, ldk, S, lds, n, k, cnt, acc, labels, own, icounts, state, scratch, bytes,
                           (cudaStream_t)stream);
}

extern "C" int pcb_kk_finalize(const int32_t* labels, const int32_t* labels_prev, const double* own, int64_t n,
                               int k, double* acc, double* cnt, double* obj_hist, long long* rep_hist,
                               long long* state, int check_convergence, double tol, void* stream) {
  if (n < 1 || k < 1 || !labels || !own || !acc || !cnt || !obj_hist || !rep_hist || !state) return PCB_EINVAL;
  if ((size_t)k * sizeof(int) > 200 * 1024) return PCB_EUNSUP;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t sm = (size_t)k * sizeof(int);
  if (sm > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kk_bookkeep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return (int)e;
  }
  const int g = (int)std::min<int64_t>((n + 255) / 256, 4L * sm_count());
  kk_bookkeep_kernel<<<g, 256, sm, st>>>(labels, labels_prev, own, n, k, acc, state);
  PCB_CHECK_LAUNCH();
  kk_finalize_kernel<<<1, 256, 0, st>>>(acc, k, n, cnt, obj_hist, rep_hist, state, check_convergence, tol);
  PCB_CHECK_LAUNCH();
  return 0;
}
