// Certified 1xTF32 screening, A-resident variant for d <= 128 (ld = 32 * NKC).
//
// Same numerics and certificate as assign_screen.cu (see its header); only the
// data movement differs.  The streaming kernel re-reads every 128-row P tile
// once per centroid tile and every centroid tile once per row tile: at c3 that
// is 61 GB of L2->SM TMA traffic per iteration (ncu, profiles/), which caps the
// tensor pipe near 65 %.  Here a CTA keeps TWO 128-row tiles (256 points) of
// P_r resident in shared memory for all centroid tiles, and streams the
// centroid tiles (BN = 128) once per 256 points:
//
//   smem   A: [2 row tiles][NKC chunks][128 x 128 B]   (NKC x 32 KB)
//          B: 4-stage ring of 128 x 128 B centroid chunks
//   TMEM   [2 buffers][2 row tiles][128 columns]  (512 columns)
//   warps  0 A producer (TMA, per K chunk, released chunk by chunk by the MMAs
//            of the previous pair so the next pair's load overlaps them)
//          3 B producer (TMA ring)
//          1 MMA issuer: per stage 2 row tiles x 4 K-steps of
//            tcgen05.mma.cta_group::1.kind::tf32 M=128 N=128 K=8
//          2 TMEM allocator
//          4-11 epilogue: warp (g, h) owns lanes 32g..32g+31 of row tile h —
//            every row belongs to one thread, no cross-warp merge.
// Traffic at c3 drops from 61 GB to 25.6 GB per iteration.
#include "pcb_common.cuh"
#include "pcb_launch.cuh"
#include "screen_common.cuh"
#include "tc_ptx.cuh"

namespace pcb {

constexpr int SR_BN = 128;
constexpr int SR_STAGES = 4;
constexpr int SR_THREADS = 384;

template <int NKC>
struct SrCfg {
  static constexpr uint32_t kTileBytes = 128 * SC_BK * 4;           // 16 KB (128 rows x 32 f32)
  static constexpr uint32_t kABytes = 2 * NKC * kTileBytes;         // resident A (2 row tiles)
  static constexpr uint32_t kBBytes = SR_BN * SC_BK * 4;            // 16 KB per B stage
  static constexpr uint32_t kBarBytes = 1024;
  static constexpr uint32_t kSmem = 1024 + kABytes + SR_STAGES * kBBytes + kBarBytes + SC_KMAX * 4;
  static_assert(kSmem <= 232448, "exceeds the 227 KB dynamic shared memory limit");
};

template <int NKC>
__global__ void __launch_bounds__(SR_THREADS, 1)
assign_screen_res_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                         const float* __restrict__ anorm, const float* __restrict__ danorm,
                         const float* __restrict__ cnorm, const float* __restrict__ bstat, int64_t n, int k,
                         int32_t* __restrict__ labels, int* __restrict__ amb_list, int* __restrict__ amb_count,
                         const long long* __restrict__ state) {
  using Cfg = SrCfg<NKC>;
  if (stopped(state)) return;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw & 1023u)) & 1023u);
  uint8_t* sA = smem;                                   // [tile][kc] 16 KB each
  uint8_t* sB = smem + Cfg::kABytes;                    // [stage] 16 KB each
  uint8_t* bar_area = sB + SR_STAGES * Cfg::kBBytes;
  uint64_t* afull = reinterpret_cast<uint64_t*>(bar_area);  // [NKC]
  uint64_t* aempty = afull + NKC;                            // [NKC]
  uint64_t* full = aempty + NKC;                             // [STAGES]
  uint64_t* empty = full + SR_STAGES;                        // [STAGES]
  uint64_t* tfull = empty + SR_STAGES;                       // [2]
  uint64_t* tempty = tfull + 2;                              // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* cprime = reinterpret_cast<float*>(bar_area + Cfg::kBarBytes);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = (k + SR_BN - 1) / SR_BN;
  const float OFF = bstat[2];
  for (int j = threadIdx.x; j < ntiles * SR_BN; j += blockDim.x)
    cprime[j] = j < k ? cnorm[j] + OFF : 3.0e38f;
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tm_a);
    ptx::prefetch_tmap(&tm_b);
    for (int c = 0; c < NKC; ++c) {
      ptx::mbar_init(&afull[c], 1);
      ptx::mbar_init(&aempty[c], 1);
    }
    for (int s = 0; s < SR_STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], 256);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t npairs = (n + 255) / 256;

  if (warp == 0) {
    // ---------------- A producer: both row tiles, chunk by chunk ----------------
    const uint64_t pol = ptx::policy_evict_first();
    int it = 0;
    for (int64_t pr = blockIdx.x; pr < npairs; pr += gridDim.x, ++it) {
      for (int c = 0; c < NKC; ++c) {
        if (it > 0) ptx::mbar_wait(&aempty[c], (uint32_t)((it - 1) & 1));
        if (ptx::elect_one()) {
          ptx::mbar_expect_tx(&afull[c], 2 * Cfg::kTileBytes);
          ptx::tma_load_2d(&tm_a, &afull[c], sA + (0 * NKC + c) * Cfg::kTileBytes, c * SC_BK, (int)(pr * 256), pol);
          ptx::tma_load_2d(&tm_a, &afull[c], sA + (1 * NKC + c) * Cfg::kTileBytes, c * SC_BK,
                           (int)(pr * 256 + 128), pol);
        }
        __syncwarp();
      }
    }
  } else if (warp == 3) {
    // ---------------- B producer: centroid chunks through the ring ----------------
    const uint64_t pol = ptx::policy_evict_last();
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t pr = blockIdx.x; pr < npairs; pr += gridDim.x) {
      for (int nt = 0; nt < ntiles; ++nt) {
        for (int c = 0; c < NKC; ++c) {
          ptx::mbar_wait(&empty[stage], phase ^ 1u);
          if (ptx::elect_one()) {
            ptx::mbar_expect_tx(&full[stage], Cfg::kBBytes);
            ptx::tma_load_2d(&tm_b, &full[stage], sB + stage * Cfg::kBBytes, c * SC_BK, nt * SR_BN, pol);
          }
          __syncwarp();
          if (++stage == SR_STAGES) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (warp-uniform loop, one elected lane issues) ----------------
    constexpr uint32_t idesc = ptx::idesc_tf32<128, SR_BN>();
    int stage = 0;
    uint32_t phase = 0;
    int abuf = 0;
    uint32_t aphase = 0;
    int it = 0;
    for (int64_t pr = blockIdx.x; pr < npairs; pr += gridDim.x, ++it) {
      for (int nt = 0; nt < ntiles; ++nt) {
        ptx::mbar_wait(&tempty[abuf], aphase ^ 1u);
        ptx::tc_fence_after();
        const uint32_t d0 = tmem + (uint32_t)(abuf * 256);
        for (int c = 0; c < NKC; ++c) {
          if (nt == 0) ptx::mbar_wait(&afull[c], (uint32_t)(it & 1));
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint64_t a0 = ptx::sdesc_k_sw128(ptx::smem_u32(sA + (0 * NKC + c) * Cfg::kTileBytes));
          const uint64_t a1 = ptx::sdesc_k_sw128(ptx::smem_u32(sA + (1 * NKC + c) * Cfg::kTileBytes));
          const uint64_t bd = ptx::sdesc_k_sw128(ptx::smem_u32(sB + stage * Cfg::kBBytes));
          if (ptx::elect_one()) {
#pragma unroll
            for (int ks = 0; ks < SC_BK / 8; ++ks) {
              const uint64_t off = (uint64_t)(ks * 8 * 4) >> 4;
              ptx::umma_tf32(d0, a0 + off, bd + off, idesc, (c | ks) != 0);
              ptx::umma_tf32(d0 + 128, a1 + off, bd + off, idesc, (c | ks) != 0);
            }
            ptx::umma_commit(&empty[stage]);
            if (nt + 1 == ntiles) ptx::umma_commit(&aempty[c]);  // A chunk free for the next pair
          }
          __syncwarp();
          if (++stage == SR_STAGES) { stage = 0; phase ^= 1u; }
        }
        if (ptx::elect_one()) ptx::umma_commit(&tfull[abuf]);
        __syncwarp();
        abuf ^= 1;
        if (abuf == 0) aphase ^= 1u;
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: warp (g, h) = lanes 32g.. of row tile h ----------------
    const int g = warp & 3, h = (warp - 4) >> 2;
    const float Bmax = bstat[0], dBmax = bstat[1];
    const float acc_rel = (float)(NKC * 4 + 2) * 9.0f * 0x1p-23f;
    const uint32_t msk = kIdxMask;
    int abuf = 0;
    uint32_t aphase = 0;
    // row norms of the next pair are loaded one pair ahead (their DRAM latency
    // otherwise stalls the first chunk of every pair)
    const int64_t r_in = h * 128 + g * 32 + lane;
    float an_nx = 0.0f, dan_nx = 0.0f;
    if (blockIdx.x < npairs) {
      const int64_t row0 = (int64_t)blockIdx.x * 256 + r_in;
      an_nx = anorm[row0 < n ? row0 : n - 1];
      dan_nx = danorm[row0 < n ? row0 : n - 1];
    }
    // c' of chunk c+1 is read from smem while chunk c is processed (ping-pong
    // register sets cpA/cpB over the 4 chunks of a tile)
    float cpA[32], cpB[32];
    for (int64_t pr = blockIdx.x; pr < npairs; pr += gridDim.x) {
      const int64_t row = pr * 256 + r_in;
      const float twoE = screen_two_e(an_nx, dan_nx, Bmax, dBmax, OFF, acc_rel);
      const float big = 64.0f / twoE;
      if (pr + gridDim.x < npairs) {
        const int64_t rn = (pr + gridDim.x) * 256 + r_in;
        an_nx = anorm[rn < n ? rn : n - 1];
        dan_nx = danorm[rn < n ? rn : n - 1];
      }
      float R1 = 3.4e38f, cnt = 0.0f;
      int r1 = 0;
      load_cprime(cpA, cprime);
      for (int nt = 0; nt < ntiles; ++nt) {
        ptx::mbar_wait(&tfull[abuf], aphase);
        ptx::tc_fence_after();
        const uint32_t taddr = tmem + ((uint32_t)(g * 32) << 16) + (uint32_t)(abuf * 256 + h * 128);
        const int c0 = nt * SR_BN;
#ifndef PCB_EXP
#define PCB_EXP 0
#endif
        static_assert(SR_BN == 128, "the ping-pong below covers 4 chunks per tile");
        float v[32];
        load_cprime(cpB, cprime + c0 + 32);
        if (PCB_EXP != 2) ptx::tmem_ld_32x32b_x32(taddr + 0, v);
        if (PCB_EXP == 0 || PCB_EXP == 3) screen_chunk_regs(v, cpA, msk, c0 + 0, twoE, big, R1, r1, cnt);
        if (PCB_EXP == 1) R1 = fminf(R1, v[0] + v[31]);
        load_cprime(cpA, cprime + c0 + 64);
        if (PCB_EXP != 2) ptx::tmem_ld_32x32b_x32(taddr + 32, v);
        if (PCB_EXP == 0 || PCB_EXP == 3) screen_chunk_regs(v, cpB, msk, c0 + 32, twoE, big, R1, r1, cnt);
        if (PCB_EXP == 1) R1 = fminf(R1, v[0] + v[31]);
        load_cprime(cpB, cprime + c0 + 96);
        if (PCB_EXP != 2) ptx::tmem_ld_32x32b_x32(taddr + 64, v);
        if (PCB_EXP == 0 || PCB_EXP == 3) screen_chunk_regs(v, cpA, msk, c0 + 64, twoE, big, R1, r1, cnt);
        if (PCB_EXP == 1) R1 = fminf(R1, v[0] + v[31]);
        if (nt + 1 < ntiles) load_cprime(cpA, cprime + c0 + 128);
        if (PCB_EXP != 2) ptx::tmem_ld_32x32b_x32(taddr + 96, v);
        if (PCB_EXP == 0 || PCB_EXP == 3) screen_chunk_regs(v, cpB, msk, c0 + 96, twoE, big, R1, r1, cnt);
        if (PCB_EXP == 1) R1 = fminf(R1, v[0] + v[31]);
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[abuf]);
        abuf ^= 1;
        if (abuf == 0) aphase ^= 1u;
      }
      if (row < n) labels[row] = r1;
      screen_append(row < n && cnt > 1.0f, row, amb_list, amb_count, lane);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc<512>(tmem);
}

template <int NKC>
static int launch_screen_res(const float* P, int64_t n, const float* C, int k, const float* an,
                             const float* dan, const float* cnorm, const float* bstat, int32_t* labels,
                             int* amb_list, int* amb_count, const long long* state, cudaStream_t st) {
  using Cfg = SrCfg<NKC>;
  CUtensorMap ta, tb;
  int rc;
  if ((rc = make_tmap_rows(&ta, P, n, NKC * SC_BK, 128))) return rc;
  if ((rc = make_tmap_rows(&tb, C, k, NKC * SC_BK, SR_BN))) return rc;
  auto kern = assign_screen_res_kernel<NKC>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::kSmem);
  if (e != cudaSuccess) return (int)e;
  const int64_t npairs = (n + 255) / 256;
  const int grid = (int)std::min<int64_t>(npairs, (int64_t)sm_count());
  kern<<<grid, SR_THREADS, Cfg::kSmem, st>>>(ta, tb, an, dan, cnorm, bstat, n, k, labels, amb_list, amb_count,
                                             state);
  PCB_CHECK_LAUNCH();
  return 0;
}

int assign_screen_resident(const float* P_r, int64_t n, int ld, const float* C_r, int k, const float* cnorm,
                           const float* anorm, const float* danorm, const float* bstat, int32_t* labels,
                           int* amb_list, int* amb_count, const long long* state, cudaStream_t st) {
  switch (ld / SC_BK) {
    case 1: return launch_screen_res<1>(P_r, n, C_r, k, anorm, danorm, cnorm, bstat, labels, amb_list, amb_count, state, st);
    case 2: return launch_screen_res<2>(P_r, n, C_r, k, anorm, danorm, cnorm, bstat, labels, amb_list, amb_count, state, st);
    case 3: return launch_screen_res<3>(P_r, n, C_r, k, anorm, danorm, cnorm, bstat, labels, amb_list, amb_count, state, st);
    case 4: return launch_screen_res<4>(P_r, n, C_r, k, anorm, danorm, cnorm, bstat, labels, amb_list, amb_count, state, st);
    default: return PCB_EUNSUP;
  }
}

}  // namespace pcb
