// Fused distance + argmin on the 5th-generation tensor cores (tcgen05), 3xTF32.
//
// Replaces clustering.py:310-311 (D = pn - 2 P C^T + cn, OpenBLAS sgemm +
// three n x k temporaries) and dense.py:56-68 (row argmin) for float32 with
// d > 32.  The n x k distance matrix never leaves the SM: the GEMM
// accumulates in TMEM and the epilogue turns each accumulator row into a
// running (min, argmin) in registers.
//
// FP32-faithful products with TF32 tensor cores (3xTF32): every operand x is
// pre-split into hi = rna_tf32(x) and lo = x - hi (exact), and
//     <p, c> ~= <p_hi, c_hi> + <p_hi, c_lo> + <p_lo, c_hi>
// (the dropped lo*lo term is ~2^-22 relative).  P is split once per fit
// (pcb_split_tf32), C once per iteration by the finalize kernel.
//
// Structure (one CTA per SM, persistent over 128-row tiles):
//   warp 0     TMA producer: per (row tile, centroid tile, 32-wide K chunk)
//              loads A_hi, A_lo (128 x 32 f32) and B_hi, B_lo (BN x 32 f32),
//              128-byte swizzled, into a STAGES-deep smem ring (mbarriers).
//   warp 1     MMA issuer (one thread): 4 K-steps x 3 products of
//              tcgen05.mma.cta_group::1.kind::tf32 M=128 N=BN K=8 per stage,
//              accumulating into one of two TMEM buffers (2 x BN columns);
//              tcgen05.commit frees smem stages and publishes accumulators.
//   warp 2     TMEM allocator.
//   warps 4-7  epilogue: tcgen05.ld 32 columns at a time (thread = row),
//              s_j = cnorm_j - 2 acc_j, running (min, lowest j), then the
//              bookkeeping of _assignment_step (labels, own distance, counts,
//              objective, changed) exactly like the FFMA kernels.
// The double-buffered accumulator lets the epilogue of centroid tile t overlap
// the MMAs of tile t+1.
#include <cudaTypedefs.h>

#include "pcb_common.cuh"
#include "pcb_launch.cuh"
#include "tc_ptx.cuh"

namespace pcb {

constexpr int TC_BM = 128;     // rows per tile (UMMA M)
constexpr int TC_BK = 32;      // f32 per 128-byte swizzle row
constexpr int TC_THREADS = 256;
constexpr int TC_HIST_MAX = 4096;
constexpr int XR_SCRATCH_ROWS = 32768;  // flagged rows whose exact pass may split the centroid range

template <int BN>
struct TcCfg {
  static constexpr int kStages = BN == 256 ? 2 : (BN == 128 ? 3 : 4);
  static constexpr uint32_t kABytes = TC_BM * TC_BK * 4;   // 16 KB
  static constexpr uint32_t kBBytes = BN * TC_BK * 4;
  static constexpr uint32_t kStageBytes = 2 * kABytes + 2 * kBBytes;
  static constexpr uint32_t kTmemCols = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                        : (2 * BN <= 256) ? 256 : 512;
  static constexpr uint32_t kBarBytes = 1024;  // barriers + tmem ptr, padded
  static constexpr uint32_t kSmem = 1024 /*align slack*/ + kStages * kStageBytes + kBarBytes +
                                    TC_HIST_MAX * 4;
};

// FLAG (the resolver of the screened variants and predict): the epilogue also
// tracks the second-best key and appends every row whose top-2 keys are within
// the rigorous error bound 2E of the 3xTF32 keys to flag_list; those rows get
// the exact argmin from exact_rows_kernel, so every label this path returns is
// the exact (f64, lowest index on ties) argmin.  Per key s_j = |c_j|^2 - 2 v_j:
//   |v_j - <p, c_j>| <= 2^-19 |p||c|   (dropped lo*lo, TF32 truncation of lo)
//                     + acc_rel |p||c| (tensor-core accumulation, 8 units of
//                                       2^-23 per MMA: 3.6x the worst single-MMA
//                                       error tests/test_gpu_mma_probe.py measures)
//   + 2^-23 (|c|^2 + 2 |p||c|)         (f32 key arithmetic, f32 norms)
// with |c| <= max_j |c_j| (cnmax = max |c_j|^2, reduced in the prologue).
template <int BN, bool FLAG = false>
__global__ void __launch_bounds__(TC_THREADS, 1)
assign_tc3xtf32_kernel(const __grid_constant__ CUtensorMap tm_ahi, const __grid_constant__ CUtensorMap tm_alo,
                       const __grid_constant__ CUtensorMap tm_bhi, const __grid_constant__ CUtensorMap tm_blo,
                       const float* __restrict__ pnorm, const float* __restrict__ cnorm, int64_t n, int k,
                       int d, int num_kc, const int32_t* __restrict__ labels_prev,
                       int32_t* __restrict__ labels, float* __restrict__ mind, double* __restrict__ acc,
                       const long long* __restrict__ state, const int* __restrict__ n_dev,
                       const int* __restrict__ row_ids = nullptr, int* __restrict__ flag_list = nullptr,
                       int* __restrict__ flag_count = nullptr) {
  using Cfg = TcCfg<BN>;
  if (stopped(state)) return;
  if (n_dev != nullptr) n = min(n, (int64_t)*n_dev);  // row count known only on the device
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw & 1023u)) & 1023u);
  uint8_t* bar_area = smem + Cfg::kStages * Cfg::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(bar_area);
  uint64_t* empty = full + Cfg::kStages;
  uint64_t* tfull = empty + Cfg::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* hist = reinterpret_cast<int*>(bar_area + Cfg::kBarBytes);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool use_hist = acc != nullptr && k <= TC_HIST_MAX;
  if (use_hist)
    for (int j = threadIdx.x; j < k; j += blockDim.x) hist[j] = 0;
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tm_ahi);
    ptx::prefetch_tmap(&tm_alo);
    ptx::prefetch_tmap(&tm_bhi);
    ptx::prefetch_tmap(&tm_blo);
    for (int s = 0; s < Cfg::kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], 128);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int64_t mtiles = (n + TC_BM - 1) / TC_BM;
  const int ntiles = (k + BN - 1) / BN;

  if (warp == 0) {
      // ---------------- TMA producer ----------------
      const uint64_t pol_a = ptx::policy_evict_first();
      const uint64_t pol_b = ptx::policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t mt = blockIdx.x; mt < mtiles; mt += gridDim.x) {
        const int y_a = (int)(mt * TC_BM);
        for (int nt = 0; nt < ntiles; ++nt) {
          for (int kc = 0; kc < num_kc; ++kc) {
            ptx::mbar_wait(&empty[stage], phase ^ 1u);
            uint8_t* st = smem + stage * Cfg::kStageBytes;
            const uint64_t pa = (nt + 1 == ntiles) ? pol_a : pol_b;  // A re-read per centroid tile
            if (ptx::elect_one()) {
              ptx::mbar_expect_tx(&full[stage], Cfg::kStageBytes);
              ptx::tma_load_2d(&tm_ahi, &full[stage], st, kc * TC_BK, y_a, pa);
              ptx::tma_load_2d(&tm_alo, &full[stage], st + Cfg::kABytes, kc * TC_BK, y_a, pa);
              ptx::tma_load_2d(&tm_bhi, &full[stage], st + 2 * Cfg::kABytes, kc * TC_BK, nt * BN, pol_b);
              ptx::tma_load_2d(&tm_blo, &full[stage], st + 2 * Cfg::kABytes + Cfg::kBBytes, kc * TC_BK,
                               nt * BN, pol_b);
            }
            __syncwarp();
            if (++stage == Cfg::kStages) { stage = 0; phase ^= 1u; }
          }
        }
      }
    
  } else if (warp == 1) {
      // ---------------- MMA issuer ----------------
      constexpr uint32_t idesc = ptx::idesc_tf32<TC_BM, BN>();
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
            const uint64_t ahi = ptx::sdesc_k_sw128(base);
            const uint64_t alo = ptx::sdesc_k_sw128(base + Cfg::kABytes);
            const uint64_t bhi = ptx::sdesc_k_sw128(base + 2 * Cfg::kABytes);
            const uint64_t blo = ptx::sdesc_k_sw128(base + 2 * Cfg::kABytes + Cfg::kBBytes);
            if (ptx::elect_one()) {
#pragma unroll
              for (int ks = 0; ks < TC_BK / 8; ++ks) {
                const uint64_t off = (uint64_t)(ks * 8 * 4) >> 4;  // 32 bytes per K=8 step
                ptx::umma_tf32(dt, ahi + off, bhi + off, idesc, (kc | ks) != 0);
                ptx::umma_tf32(dt, ahi + off, blo + off, idesc, 1u);
                ptx::umma_tf32(dt, alo + off, bhi + off, idesc, 1u);
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
    // ---------------- epilogue ----------------
    const int ew = warp - 4;  // TMEM lane group ew*32 .. ew*32+31
    const int r_in_tile = ew * 32 + lane;
    int abuf = 0;
    uint32_t aphase = 0;
    long long chg = 0;
    float cnmax = 0.0f, acc_rel = 0.0f;
    if (FLAG) {
      for (int j = r_in_tile; j < k; j += 128) cnmax = fmaxf(cnmax, cnorm[j]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) cnmax = fmaxf(cnmax, __shfl_xor_sync(0xffffffffu, cnmax, o));
      if (lane == 0) hist[ew] = __float_as_int(cnmax);
      ptx::named_bar_sync(1, 128);
      cnmax = fmaxf(fmaxf(__int_as_float(hist[0]), __int_as_float(hist[1])),
                    fmaxf(__int_as_float(hist[2]), __int_as_float(hist[3])));
      acc_rel = (float)(3 * 4 * num_kc + 3) * 0x1p-20f;  // 3 MMAs per K = 8 step, 4 steps per chunk
    }
    for (int64_t mt = blockIdx.x; mt < mtiles; mt += gridDim.x) {
      float best = INFINITY, second = INFINITY;
      int bj = 0;
      for (int nt = 0; nt < ntiles; ++nt) {
        ptx::mbar_wait(&tfull[abuf], aphase);
        ptx::tc_fence_after();
        const uint32_t taddr = tmem + ((uint32_t)(ew * 32) << 16) + (uint32_t)(abuf * BN);
        const int jbase = nt * BN;
#pragma unroll 1
        for (int cb = 0; cb < BN; cb += 32) {
          float v[32];
          ptx::tmem_ld_32x32b_x32(taddr + cb, v);
          const int j0 = jbase + cb;
          if (j0 + 32 <= k) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float s = fmaf(-2.0f, v[i], __ldg(&cnorm[j0 + i]));
              if (FLAG) second = fminf(second, fmaxf(s, best));
              if (s < best) { best = s; bj = j0 + i; }
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              if (j0 + i < k) {
                const float s = fmaf(-2.0f, v[i], __ldg(&cnorm[j0 + i]));
                if (FLAG) second = fminf(second, fmaxf(s, best));
                if (s < best) { best = s; bj = j0 + i; }
              }
            }
          }
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[abuf]);
        abuf ^= 1;
        if (abuf == 0) aphase ^= 1u;
      }
      const int64_t row = mt * TC_BM + r_in_tile;
      if (FLAG) {
        bool flag = false;
        if (row < n) {
          const float pn = pnorm[row_ids != nullptr ? (int64_t)row_ids[row] : row];
          const float A = sqrtf(pn) * sqrtf(cnmax) * 1.0001f;  // >= |p| max|c|
          const float E = (2.0f * (0x1p-19f + acc_rel) * A + 0x1p-23f * (cnmax + 2.0f * A)) * 1.01f;
          flag = !(second - best > 2.0f * E);  // NaN keys are flagged too
        }
        const unsigned fm = __ballot_sync(0xffffffffu, flag);
        if (fm) {
          int b = 0;
          if (lane == 0) b = atomicAdd(flag_count, __popc(fm));
          b = __shfl_sync(0xffffffffu, b, 0);
          if (flag) flag_list[b + __popc(fm & ((1u << lane) - 1u))] = (int)row;
        }
      }
      if (row < n) {
        const float own = pnorm[row] + best;
        labels[row] = bj;
        if (mind) mind[row] = own;
        if (acc) {
          if (labels_prev) chg += (labels_prev[row] != bj);
          if (use_hist) atomicAdd(&hist[bj], 1);
          else atomicAdd(&acc[(int64_t)k * d + bj], 1.0);
        }
        if (state != nullptr && !isfinite(own))
          atomicExch((unsigned long long*)&state[kNanFlag], 1ull);
      }
    }
    if (acc) {
      chg = warp_sum(chg);
      if (lane == 0) atomicAdd(&acc[(int64_t)k * d + k + 1], (double)chg);
      ptx::named_bar_sync(1, 128);
      if (use_hist)
        for (int j = r_in_tile; j < k; j += 128)
          if (hist[j]) atomicAdd(&acc[(int64_t)k * d + j], (double)hist[j]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc<Cfg::kTmemCols>(tmem);
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
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

// 2-D row-major f32 matrix (rows x ld), box = 32 columns x box_rows rows, 128B swizzle.
static int make_tmap(CUtensorMap* m, const float* base, int64_t rows, int ld, int box_rows) {
  auto enc = tmap_encoder();
  if (!enc) return PCB_ENODEV;
  cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
  cuuint32_t box[2] = {(cuuint32_t)TC_BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : PCB_EINVAL;
}

template <int BN>
static int launch_tc(const float* phi, const float* plo, int ld, const float* pnorm, int64_t n, int d,
                     const float* chi, const float* clo, const float* cnorm, int k, const int32_t* lp,
                     int32_t* lab, float* mind, double* acc, const long long* state, cudaStream_t st,
                     const int* n_dev = nullptr, const int* row_ids = nullptr, int* flag_list = nullptr,
                     int* flag_count = nullptr) {
  using Cfg = TcCfg<BN>;
  CUtensorMap ta_hi, ta_lo, tb_hi, tb_lo;
  int rc;
  if ((rc = make_tmap(&ta_hi, phi, n, ld, TC_BM))) return rc;
  if ((rc = make_tmap(&ta_lo, plo, n, ld, TC_BM))) return rc;
  if ((rc = make_tmap(&tb_hi, chi, k, ld, BN))) return rc;
  if ((rc = make_tmap(&tb_lo, clo, k, ld, BN))) return rc;
  auto kern = flag_list != nullptr ? assign_tc3xtf32_kernel<BN, true> : assign_tc3xtf32_kernel<BN, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::kSmem);
  if (e != cudaSuccess) return (int)e;
  const int64_t mtiles = (n + TC_BM - 1) / TC_BM;
  const int grid = (int)std::min<int64_t>(mtiles, (int64_t)sm_count());
  kern<<<grid, TC_THREADS, Cfg::kSmem, st>>>(ta_hi, ta_lo, tb_hi, tb_lo, pnorm, cnorm, n, k, d, ld / TC_BK, lp,
                                              lab, mind, acc, state, n_dev, row_ids, flag_list, flag_count);
  PCB_CHECK_LAUNCH();
  return 0;
}

// 3xTF32 assignment of a row subset whose count lives on the device (the
// ambiguous rows of the screened kernel, compacted by gather_split_rows).
int assign_tc3xtf32_devcount(const float* phi, const float* plo, int ld, const float* pnorm, int64_t cap,
                             int d, const float* chi, const float* clo, const float* cnorm, int k,
                             int32_t* lab, const int* n_dev, const long long* state, cudaStream_t st,
                             const int* row_ids, int* flag_list, int* flag_count) {
  if (k > 128)
    return launch_tc<256>(phi, plo, ld, pnorm, cap, d, chi, clo, cnorm, k, nullptr, lab, nullptr, nullptr,
                          state, st, n_dev, row_ids, flag_list, flag_count);
  if (k > 64)
    return launch_tc<128>(phi, plo, ld, pnorm, cap, d, chi, clo, cnorm, k, nullptr, lab, nullptr, nullptr,
                          state, st, n_dev, row_ids, flag_list, flag_count);
  return launch_tc<64>(phi, plo, ld, pnorm, cap, d, chi, clo, cnorm, k, nullptr, lab, nullptr, nullptr, state,
                       st, n_dev, row_ids, flag_list, flag_count);
}

// ---------------------------------------------------------------------------
// Exact argmin (dense.py:56-68) over all k centroids for the rows the 3xTF32
// pass flagged (flag_list; row r of P is P[row_ids[r]], label -> out[r]):
// sum_t (p_t - c_t)^2 in f64 for every (row, centroid) pair, lowest index on
// ties.  32 rows per block, centroids in tiles of 64 and columns in chunks of
// 32 staged in shared memory (f32, converted exactly), each thread 4 rows x
// 4 centroids with sequential f64 sums.  Few flagged rows (steady state:
// ~1e3) would leave most SMs idle, so the centroid range is split over
// gridDim.y segments (chosen on the device from the row count) whose partial
// argmins exact_merge_kernel combines; with one segment the block writes the
// labels itself.  (f32 sums with a rigorous margin were tried first: at the
// cold start every flagged row's margin is thinner than the f32 error of
// distances ~4e3, so everything fell through to an f64 pass anyway.)
// ---------------------------------------------------------------------------
constexpr int XR_R = 32, XR_C = 64, XR_K = 32, XR_SEG = 16;

struct ExactScratch {
  int seg;                         // centroid segments of this launch
  int pad;
  double dmin[XR_SEG * XR_SCRATCH_ROWS];
  int bj[XR_SEG * XR_SCRATCH_ROWS];
};

__device__ __forceinline__ int exact_segments(int cnt, int nblk_x, int k) {
  const int nrb = (cnt + XR_R - 1) / XR_R;
  if (nrb == 0 || nrb * XR_R > XR_SCRATCH_ROWS) return 1;
  int seg = (nblk_x * 2) / nrb;  // ~2 blocks per SM in flight
  seg = seg < 1 ? 1 : (seg > XR_SEG ? XR_SEG : seg);
  const int maxseg = (k + XR_C - 1) / XR_C;
  return seg < maxseg ? seg : maxseg;
}

__device__ __forceinline__ void argmin_take(double& v, int& j, double v2, int j2) {
  if (v2 < v || (v2 == v && j2 < j)) { v = v2; j = j2; }
}

__global__ void __launch_bounds__(128)
exact_tiled_kernel(const float* __restrict__ P, int d, const float* __restrict__ C, int k,
                   const int* __restrict__ flag_list, const int* __restrict__ flag_count,
                   const int* __restrict__ row_ids, int32_t* __restrict__ out, ExactScratch* __restrict__ sc,
                   const long long* __restrict__ state) {
  if (stopped(state)) return;
  // f64 tiles, converted once per element at staging (not once per use in the
  // inner loop); rows padded by 2 doubles against bank conflicts of the
  // transposing stores, 16-byte aligned for the double2 reads
  __shared__ __align__(16) double sP[XR_K][XR_R + 2];
  __shared__ __align__(16) double sC[XR_K][XR_C + 2];
  __shared__ int64_t srow[XR_R];
  __shared__ int sidx[XR_R];
  const int cnt = *flag_count;
  const int seg = exact_segments(cnt, gridDim.x, k);
  if (blockIdx.x == 0 && threadIdx.x == 0) sc->seg = seg;
  const int ctiles = (k + XR_C - 1) / XR_C;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  // work items (row block, centroid segment) over a 1-D grid: a launch sized for
  // the cold start's ~1e5 flagged rows costs little when only ~1e2 are flagged
  const int nrb = (cnt + XR_R - 1) / XR_R;
  for (int item = blockIdx.x; item < nrb * seg; item += gridDim.x) {
    const int sg = item % seg, rb = (item / seg) * XR_R;
    const int t_lo = (int)((int64_t)ctiles * sg / seg), t_hi = (int)((int64_t)ctiles * (sg + 1) / seg);
    __syncthreads();
    if (tid < XR_R) {
      const int q = rb + tid;
      const int r = q < cnt ? flag_list[q] : -1;
      sidx[tid] = r;
      srow[tid] = r < 0 ? -1 : (row_ids != nullptr ? (int64_t)row_ids[r] : (int64_t)r);
    }
    double best[4];
    int bj[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) { best[i] = 1.0e308; bj[i] = 0x7fffffff; }
    for (int ct = t_lo; ct < t_hi; ++ct) {
      const int c0 = ct * XR_C;
      double acc[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
      for (int k0 = 0; k0 < d; k0 += XR_K) {
        __syncthreads();
        for (int e = tid; e < XR_R * XR_K; e += 128) {  // row-contiguous reads
          const int r = e / XR_K, kk = e % XR_K;
          const int64_t pr = srow[r];
          sP[kk][r] = (pr >= 0 && k0 + kk < d) ? (double)__ldg(P + pr * d + k0 + kk) : 0.0;
        }
        for (int e = tid; e < XR_C * XR_K; e += 128) {
          const int c = e / XR_K, kk = e % XR_K;
          sC[kk][c] = (c0 + c < k && k0 + kk < d) ? (double)__ldg(C + (int64_t)(c0 + c) * d + k0 + kk) : 0.0;
        }
        __syncthreads();
#pragma unroll 4
        for (int kk = 0; kk < XR_K; ++kk) {
          const double2 a0 = *reinterpret_cast<const double2*>(&sP[kk][ty * 4]);
          const double2 a1 = *reinterpret_cast<const double2*>(&sP[kk][ty * 4 + 2]);
          const double2 b0 = *reinterpret_cast<const double2*>(&sC[kk][tx * 4]);
          const double2 b1 = *reinterpret_cast<const double2*>(&sC[kk][tx * 4 + 2]);
          const double av[4] = {a0.x, a0.y, a1.x, a1.y}, bv[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const double e = av[i] - bv[j];
              acc[i][j] = fma(e, e, acc[i][j]);
            }
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int cj = c0 + tx * 4 + j;
        if (cj < k) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (acc[i][j] < best[i]) { best[i] = acc[i][j]; bj[i] = cj; }  // ascending cj: ties keep the lowest
        }
      }
    }
    // merge over the 16 threads of each row group (lanes ty*16 .. ty*16+15 of a warp)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, best[i], o);
        const int j2 = __shfl_xor_sync(0xffffffffu, bj[i], o);
        argmin_take(best[i], bj[i], v2, j2);
      }
    }
    if (tx == 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int q = rb + ty * 4 + i;
        const int r = sidx[ty * 4 + i];
        if (r < 0) continue;
        if (seg > 1) {
          sc->dmin[sg * XR_SCRATCH_ROWS + q] = best[i];
          sc->bj[sg * XR_SCRATCH_ROWS + q] = bj[i];
        } else {
          out[r] = bj[i];
        }
      }
    }
  }
}

// Several centroid segments: combine their partial argmins per flagged row.
__global__ void __launch_bounds__(256)
exact_merge_kernel(const int* __restrict__ flag_list, const int* __restrict__ flag_count, int32_t* __restrict__ out,
                   const ExactScratch* __restrict__ sc, const long long* __restrict__ state) {
  if (stopped(state)) return;
  const int cnt = *flag_count;
  const int seg = ((volatile const ExactScratch*)sc)->seg;
  if (seg <= 1) return;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < cnt; q += gridDim.x * blockDim.x) {
    double v = sc->dmin[q];
    int j = sc->bj[q];
    for (int s = 1; s < seg; ++s) argmin_take(v, j, sc->dmin[s * XR_SCRATCH_ROWS + q], sc->bj[s * XR_SCRATCH_ROWS + q]);
    out[flag_list[q]] = j;
  }
}

int exact_rows(const float* P, int d, const float* C, int k, const int* flag_list, const int* flag_count,
               const int* row_ids, int32_t* out, void* scratch, const long long* state, cudaStream_t st) {
  ExactScratch* sc = (ExactScratch*)scratch;
  const int gx = sm_count() * 4;
  exact_tiled_kernel<<<gx, 128, 0, st>>>(P, d, C, k, flag_list, flag_count, row_ids, out, sc, state);
  PCB_CHECK_LAUNCH();
  exact_merge_kernel<<<sm_count(), 256, 0, st>>>(flag_list, flag_count, out, sc, state);
  PCB_CHECK_LAUNCH();
  return 0;
}

int64_t exact_scratch_bytes() { return (int64_t)sizeof(ExactScratch); }

}  // namespace pcb

extern "C" int pcb_assign_tc_f32(const float* P_hi, const float* P_lo, int ld, const float* pnorm, int64_t n,
                                 int d, const float* C_hi, const float* C_lo, const float* cnorm, int k,
                                 const int32_t* labels_prev, int32_t* labels, float* mind, double* acc,
                                 const long long* state, void* stream) {
  if (n < 1 || d < 1 || k < 1 || ld < d || ld % pcb::TC_BK != 0 || !P_hi || !P_lo || !C_hi || !C_lo ||
      !pnorm || !cnorm || !labels)
    return PCB_EINVAL;
  if (n > INT32_MAX) return PCB_EUNSUP;  // TMA coordinates are 32-bit
  cudaStream_t st = (cudaStream_t)stream;
  if (k > 128)
    return pcb::launch_tc<256>(P_hi, P_lo, ld, pnorm, n, d, C_hi, C_lo, cnorm, k, labels_prev, labels, mind,
                               acc, state, st);
  if (k > 64)
    return pcb::launch_tc<128>(P_hi, P_lo, ld, pnorm, n, d, C_hi, C_lo, cnorm, k, labels_prev, labels, mind,
                               acc, state, st);
  return pcb::launch_tc<64>(P_hi, P_lo, ld, pnorm, n, d, C_hi, C_lo, cnorm, k, labels_prev, labels, mind,
                            acc, state, st);
}
