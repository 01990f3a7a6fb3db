// Certified 1xTF32 screening on CTA pairs (tcgen05 cta_group::2), d <= 128.
//
// Same certificate and epilogue as assign_screen.cu / assign_screen_res.cu.
// The single-SM resident kernel is limited by shared-memory operand bandwidth:
// an M=128 x N=128 x K=8 TF32 MMA reads 4 KB of A and 4 KB of B from smem every
// 64 cycles (128 B/clk/SM), which together with the TMA writes caps the tensor
// pipe near 70 % (ncu, profiles/).  Here two CTAs on an SM pair issue
// M=256 x N=256 MMAs (cta_group::2): each CTA supplies its own 128 rows of A and
// one half (128 centroid rows) of B, so per SM the MMA reads 8 KB per 128
// cycles (64 B/clk) and the TMA writes half the B tile.
//
//   per CTA smem  A: this CTA's 128-row tile of P_r, all K chunks (resident)
//                 B: 4-stage ring of 128 x 32 f32 centroid chunks (its half)
//   per CTA TMEM  2 accumulators x 256 columns (its 128 rows of the M=256 tile)
//   warps  0 A producer, 3 B producer (both CTAs; 2-SM TMA signals the leader)
//          1 MMA issuer (leader CTA only), commits multicast to both CTAs
//          2 TMEM allocator (cta_group::2)
//          4-11 epilogue (both CTAs): lane group g, column half h; the
//               accumulator-empty arrivals go to the leader's barrier
#include "pcb_common.cuh"
#include "pcb_launch.cuh"
#include "screen_common.cuh"
#include "tc_ptx.cuh"

namespace pcb {

constexpr int S2_BN = 256;       // MMA N (centroids per tile, 128 per CTA)
#ifndef PCB_S2_STAGES
#define PCB_S2_STAGES 8
#endif
constexpr int S2_STAGES = PCB_S2_STAGES;
constexpr int S2_THREADS = 384;

template <int NKC>
struct S2Cfg {
  static constexpr uint32_t kTileBytes = 128 * SC_BK * 4;  // 16 KB
  static constexpr uint32_t kABytes = NKC * kTileBytes;
  static constexpr uint32_t kBBytes = kTileBytes;
  static constexpr uint32_t kBarBytes = 4096;
  static constexpr uint32_t kSmem = 1024 + kABytes + S2_STAGES * kBBytes + kBarBytes + SC_KMAX * 4;
  static_assert(kSmem <= 232448, "exceeds the 227 KB dynamic shared memory limit");
};

template <int NKC>
__global__ void __launch_bounds__(S2_THREADS, 1)
assign_screen_2sm_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                         const float* __restrict__ anorm, const float* __restrict__ danorm,
                         const float* __restrict__ cnorm, const float* __restrict__ bstat, int64_t n, int k,
                         int32_t* __restrict__ labels, int* __restrict__ amb_list, int* __restrict__ amb_count,
                         const long long* __restrict__ state) {
  using Cfg = S2Cfg<NKC>;
  if (stopped(state)) return;  // same decision in both CTAs of the pair
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + Cfg::kABytes;
  uint8_t* bar_area = sB + S2_STAGES * Cfg::kBBytes;
  uint64_t* afull = reinterpret_cast<uint64_t*>(bar_area);  // [NKC]  (leader's are used)
  uint64_t* aempty = afull + NKC;                            // [NKC]
  uint64_t* full = aempty + NKC;                             // [STAGES] (leader's are used)
  uint64_t* empty = full + S2_STAGES;                        // [STAGES]
  uint64_t* tfull = empty + S2_STAGES;                       // [2]
  uint64_t* tempty = tfull + 2;                              // [2]  (leader's are used)
  uint64_t* xwritten = tempty + 2;                           // [4][2]
  uint64_t* xreleased = xwritten + 8;                        // [4][2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xreleased + 8);
  float* xchg = reinterpret_cast<float*>(tmem_slot + 4);     // [2][128][3]
  float* cprime = reinterpret_cast<float*>(bar_area + Cfg::kBarBytes);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int ntiles = (k + S2_BN - 1) / S2_BN;
  const float OFF = bstat[2];
  for (int j = threadIdx.x; j < ntiles * S2_BN; j += blockDim.x)
    cprime[j] = j < k ? cnorm[j] + OFF : 3.0e38f;
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tm_a);
    ptx::prefetch_tmap(&tm_b);
    for (int c = 0; c < NKC; ++c) {
      ptx::mbar_init(&afull[c], 1);
      ptx::mbar_init(&aempty[c], 1);
    }
    for (int s = 0; s < S2_STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], 2 * 256);  // both CTAs' epilogue threads
    }
    for (int b = 0; b < 8; ++b) {
      ptx::mbar_init(&xwritten[b], 32);
      ptx::mbar_init(&xreleased[b], 32);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc_2sm<512>(tmem_slot);
  ptx::tc_fence_before();
  ptx::cluster_sync();  // both CTAs' barriers exist before any remote arrive / 2-SM TMA
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t ntile256 = (n + 255) / 256;
  const int64_t c0 = ptx::cluster_id_x(), nc = ptx::nclusters_x();

  if (warp == 0) {
    // ---------------- A producer (both CTAs): this CTA's 128 rows ----------------
    const uint64_t pol = ptx::policy_evict_first();
    int it = 0;
    for (int64_t t = c0; t < ntile256; t += nc, ++it) {
      for (int c = 0; c < NKC; ++c) {
        if (it > 0) ptx::mbar_wait(&aempty[c], (uint32_t)((it - 1) & 1));
        if (ptx::elect_one()) {
          if (leader) ptx::mbar_expect_tx(&afull[c], 2 * Cfg::kTileBytes);
          ptx::tma_load_2d_2sm(&tm_a, &afull[c], sA + c * Cfg::kTileBytes, c * SC_BK, (int)(t * 256 + rank * 128),
                               pol);
        }
        __syncwarp();
      }
    }
  } else if (warp == 3) {
    // ---------------- B producer (both CTAs): this CTA's half of each tile ----------------
    const uint64_t pol = ptx::policy_evict_last();
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t t = c0; t < ntile256; t += nc) {
      for (int nt = 0; nt < ntiles; ++nt) {
        for (int c = 0; c < NKC; ++c) {
          ptx::mbar_wait(&empty[stage], phase ^ 1u);
          if (ptx::elect_one()) {
            if (leader) ptx::mbar_expect_tx(&full[stage], 2 * Cfg::kBBytes);
            ptx::tma_load_2d_2sm(&tm_b, &full[stage], sB + stage * Cfg::kBBytes, c * SC_BK,
                                 nt * S2_BN + (int)rank * 128, pol);
          }
          __syncwarp();
          if (++stage == S2_STAGES) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ---------------- MMA issuer (leader CTA): M=256 x N=256 across the pair ----------------
      constexpr uint32_t idesc = ptx::idesc_tf32<256, S2_BN>();
      int stage = 0;
      uint32_t phase = 0;
      int abuf = 0;
      uint32_t aphase = 0;
      int it = 0;
      for (int64_t t = c0; t < ntile256; t += nc, ++it) {
        for (int nt = 0; nt < ntiles; ++nt) {
          ptx::mbar_wait(&tempty[abuf], aphase ^ 1u);
          ptx::tc_fence_after();
          const uint32_t dt = tmem + (uint32_t)(abuf * S2_BN);
          for (int c = 0; c < NKC; ++c) {
            if (nt == 0) ptx::mbar_wait(&afull[c], (uint32_t)(it & 1));
            ptx::mbar_wait(&full[stage], phase);
            ptx::tc_fence_after();
            const uint64_t ad = ptx::sdesc_k_sw128(ptx::smem_u32(sA + c * Cfg::kTileBytes));
            const uint64_t bd = ptx::sdesc_k_sw128(ptx::smem_u32(sB + stage * Cfg::kBBytes));
            if (ptx::elect_one()) {
#pragma unroll
              for (int ks = 0; ks < SC_BK / 8; ++ks) {
                const uint64_t off = (uint64_t)(ks * 8 * 4) >> 4;
                ptx::umma_tf32_2sm(dt, ad + off, bd + off, idesc, (c | ks) != 0);
              }
              ptx::umma_commit_2sm(&empty[stage]);
              if (nt + 1 == ntiles) ptx::umma_commit_2sm(&aempty[c]);
            }
            __syncwarp();
            if (++stage == S2_STAGES) { stage = 0; phase ^= 1u; }
          }
          if (ptx::elect_one()) ptx::umma_commit_2sm(&tfull[abuf]);
          __syncwarp();
          abuf ^= 1;
          if (abuf == 0) aphase ^= 1u;
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (both CTAs): 128 rows x 256 columns per tile ----------------
    const int g = warp & 3, h = (warp - 4) >> 2;
    const int r_in_tile = g * 32 + lane;
    const float Bmax = bstat[0], dBmax = bstat[1];
    const float acc_rel = (float)(NKC * 4 + 2) * 9.0f * 0x1p-23f;
    const uint32_t msk = kIdxMask;
    int abuf = 0;
    uint32_t aphase = 0;
    int tile_it = 0;
    for (int64_t t = c0; t < ntile256; t += nc) {
      const int64_t row = t * 256 + rank * 128 + r_in_tile;
      const int64_t rr = row < n ? row : n - 1;
      const float twoE = screen_two_e(anorm[rr], danorm[rr], Bmax, dBmax, OFF, acc_rel);
      const float big = 64.0f / twoE;
      float R1 = 3.4e38f, cnt = 0.0f;
      int r1 = 0;
      for (int nt = 0; nt < ntiles; ++nt) {
        ptx::mbar_wait(&tfull[abuf], aphase);
        ptx::tc_fence_after();
        const uint32_t taddr = tmem + ((uint32_t)(g * 32) << 16) + (uint32_t)(abuf * S2_BN);
#ifndef PCB_EXP
#define PCB_EXP 0
#endif
#pragma unroll 1
        for (int cb = h * 32; cb < S2_BN; cb += 64) {
          float v[32];
          if (PCB_EXP != 2) ptx::tmem_ld_32x32b_x32(taddr + cb, v);
          if (PCB_EXP == 0 || PCB_EXP == 3) screen_chunk(v, cprime + nt * S2_BN + cb, msk, nt * S2_BN + cb, twoE, big, R1, r1, cnt);
          if (PCB_EXP == 1) R1 = fminf(R1, v[0] + v[31]);
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive_remote(&tempty[abuf], 0);  // the leader's MMA waits on both CTAs
        abuf ^= 1;
        if (abuf == 0) aphase ^= 1u;
      }
      // merge the two column halves of every row (see assign_screen.cu)
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
        screen_append(amb && row < n, row, amb_list, amb_count, lane);
      }
      ++tile_it;
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc_2sm<512>(tmem);
}

template <int NKC>
static int launch_screen_2sm(const float* P, int64_t n, const float* C, int k, const float* an, const float* dan,
                             const float* cnorm, const float* bstat, int32_t* labels, int* amb_list,
                             int* amb_count, const long long* state, cudaStream_t st) {
  using Cfg = S2Cfg<NKC>;
  CUtensorMap ta, tb;
  int rc;
  if ((rc = make_tmap_rows(&ta, P, n, NKC * SC_BK, 128))) return rc;
  if ((rc = make_tmap_rows(&tb, C, k, NKC * SC_BK, 128))) return rc;
  auto kern = assign_screen_2sm_kernel<NKC>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::kSmem);
  if (e != cudaSuccess) return (int)e;
  const int64_t tiles = (n + 255) / 256;
  int clusters = (int)std::min<int64_t>(tiles, (int64_t)(sm_count() / 2));
  if (clusters < 1) clusters = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * clusters);
  cfg.blockDim = dim3(S2_THREADS);
  cfg.dynamicSmemBytes = Cfg::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, ta, tb, an, dan, cnorm, bstat, n, k, labels, amb_list, amb_count, state);
  return (int)e;
}

int assign_screen_pair(const float* P_r, int64_t n, int ld, const float* C_r, int k, const float* cnorm,
                       const float* anorm, const float* danorm, const float* bstat, int32_t* labels, int* amb_list,
                       int* amb_count, const long long* state, cudaStream_t st) {
  switch (ld / SC_BK) {
    case 1: return launch_screen_2sm<1>(P_r, n, C_r, k, anorm, danorm, cnorm, bstat, labels, amb_list, amb_count, state, st);
    case 2: return launch_screen_2sm<2>(P_r, n, C_r, k, anorm, danorm, cnorm, bstat, labels, amb_list, amb_count, state, st);
    case 3: return launch_screen_2sm<3>(P_r, n, C_r, k, anorm, danorm, cnorm, bstat, labels, amb_list, amb_count, state, st);
    case 4: return launch_screen_2sm<4>(P_r, n, C_r, k, anorm, danorm, cnorm, bstat, labels, amb_list, amb_count, state, st);
    default: return PCB_EUNSUP;
  }
}

}  // namespace pcb
