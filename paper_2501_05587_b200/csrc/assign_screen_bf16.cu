// Certified BF16 screening (variant "bf16s"), A-resident, d <= 256.
//
// Same certificate as the TF32 screen (assign_screen.cu header), with one
// BF16 tensor-core pass (tcgen05.mma kind::f16, twice the TF32 rate, half the
// operand bytes) over RN-rounded operands p~ = bf16(p), c~ = bf16(c):
//
//   |<p,c> - <p~,c~>| <= |dp||c~| + |p~||dc| + |dp||dc| + acc
//
// (dp = p - p~, dc = c - c~ exact residual norms per row / per centroid; acc
// bounds the tensor core's f32 accumulation: BF16 products are exact in f32,
// each K=16 MMA adds at most (16 + 1) roundings relative to the running sum of
// |products|, charged here as (#MMA + 2) * 2^-19 of |p~||c~|, 16x the f32 unit
// roundoff per MMA).  Rows whose second-best key is within 2E of the best are
// ambiguous; unlike the TF32 screen they are resolved in two cheap steps:
//
//   pass 1 (CAND = false) all rows: labels of certified rows; ambiguous rows
//          are appended with their threshold thr = R1 + 2E (+ packing slack)
//   pass 2 (CAND = true)  the ambiguous rows only (gathered into a compact
//          copy): the same MMA recomputes every key and the epilogue emits the
//          candidate columns {j : key_j <= thr} (the exact argmin is among them:
//          key_j* <= exact_j* + E <= exact_jmin + E <= R1 + 2E)
//   exact  (pcb_screen_exact) one warp per ambiguous row evaluates
//          sum_t (p_t - c_jt)^2 in f64 for its <= SB_NCAND candidates and takes
//          the smallest (lowest index on ties, dense.py:56-68); rows with more
//          candidates (e.g. right after a random-label init, when every
//          centroid sits near the global mean) go to the 3xTF32 resolver.
//
// Layout (per CTA, 384 threads, one CTA per SM):
//   smem   A: [2 row tiles][NKC chunks][128 rows x 128 B]  (64 BF16 per row chunk)
//          B: 4-stage ring of [128 centroids x 128 B] chunks
//   TMEM   [2 buffers][2 row tiles][128 columns] = 512 columns
//   warps  0 A producer, 3 B producer, 1 MMA issuer (M=128 N=128 K=16),
//          2 TMEM allocator, 4-11 epilogue (warp (g, h): lanes 32g.. of tile h)
#include <cuda_bf16.h>
#include <cstdlib>
#include <cudaTypedefs.h>

#include "pcb_common.cuh"
#include "pcb_launch.cuh"
#include "screen_common.cuh"

#include "tc_ptx.cuh"

namespace pcb {

constexpr int SB_BN = 128;
#ifndef PCB_EPI_X4
#define PCB_EPI_X4 1
#endif
#ifndef PCB_SB_STAGES
#define PCB_SB_STAGES 4
#endif
constexpr int SB_STAGES = PCB_SB_STAGES;  // centroid-chunk ring depth (capped by shared memory)
#ifndef PCB_REGS_LOW
#define PCB_REGS_LOW 96
#endif
constexpr int SB_THREADS = 384;
constexpr int SB_BKE = 64;      // BF16 elements per 128-byte swizzle row
constexpr int SB_NCAND = 64;    // candidate slots per ambiguous row (pass 2)
constexpr int SB_AUG = 16;      // augmented K columns per centroid: |c|^2 + OFF as 3 BF16 pieces, 13 zeros
constexpr int SB_KPAD = 256;    // centroid rows of C_b / C_aug are padded to a multiple of the widest tile

// W = false: centroid tiles of 128 (MMA N = 128), TMEM = 2 buffers x 2 row
//            tiles x 128 columns, 8 epilogue warps on both row tiles.
// W = true  (d <= 128): centroid tiles of 256 (MMA N = 256: 96 instead of 128
//            bytes of shared-memory operands per cycle at full MMA rate), TMEM =
//            one 256-column accumulator per row tile; the MMAs of the two row
//            tiles alternate, so each row tile's 4 epilogue warps (full rows,
//            8 chunks per tile) overlap the other row tile's MMAs.
// RT = row tiles of 128 resident per CTA (2; 1 for rows longer than 4 chunks,
// whose operand tiles would not fit twice).
// CB = bytes per operand row chunk: 128 (SWIZZLE_128B) or 64 (SWIZZLE_64B,
// E4M3 rows of d <= 64, so they are not half padding).
template <int NKC, bool W = false, int RT = 2, int CB = 128>
struct SbCfg {
  static constexpr int kChunkBytes = CB;
  static constexpr int kKSteps = CB / 32;                           // MMAs per chunk (32 bytes of each row)
  static constexpr int kRows = 128 * RT;                            // rows per "pair"
  static constexpr int kBN = W ? 256 : 128;                         // centroids per tile
  static constexpr int kChunks = kBN / 32;                          // epilogue chunks per tile
  static constexpr uint32_t kTileBytes = 128 * CB;                  // 128 rows x CB bytes
  // resident A (2 row tiles), double-buffered across row pairs when it fits
  // (the next pair's rows load while the current pair's MMAs run)
  static constexpr int kAStages = (!W && RT * NKC <= 4) ? 2 : 1;
  static constexpr uint32_t kAPair = RT * NKC * kTileBytes;
  static constexpr uint32_t kABytes = kAStages * kAPair;
  static constexpr uint32_t kBBytes = kBN * CB;                     // centroid chunk per B stage
  static constexpr uint32_t kAugBytes = kBN * 32;                   // + the K=16 augmented columns
  static constexpr uint32_t kStageB = kBBytes + kAugBytes;          // 1024-aligned
  static constexpr uint32_t kAAug = 128 * 32;                       // constant A columns [1 1 1 0 ..]
  static constexpr uint32_t kBarBytes = 1024;
  static constexpr int kStagesFit = (int)((232448u - 1024u - kABytes - kAAug - kBarBytes) / kStageB);
  static constexpr int kStages = W ? 3 : (SB_STAGES < kStagesFit ? SB_STAGES : kStagesFit);
  static constexpr uint32_t kSmem = 1024 + kABytes + kStages * kStageB + kAAug + kBarBytes;
  static_assert(kSmem <= 232448, "exceeds the 227 KB dynamic shared memory limit");
  // setmaxnreg split of the CTA's registers: producer / MMA warpgroup
  // (kRegsLow) and the two epilogue warpgroups (kRegsHigh).  setmaxnreg.inc
  // only draws on what the CTA was launched with (384 x 168, the
  // __launch_bounds__ cap; checked at launch): 128 low + 256 high <= 64512.
  static constexpr int kLaunchRegs = 168;
  static constexpr int kRegsLow = PCB_REGS_LOW;
  static constexpr int kRegsHigh = (SB_THREADS * kLaunchRegs - 128 * kRegsLow) / 256 / 8 * 8;
  static_assert(!W || NKC <= 2, "the wide layout keeps a whole tile's chunks in the ring");
  static_assert(!W || RT == 2, "the wide layout alternates two row tiles");
};

// First centroid column of a row pair: the previous label of the pair's
// middle row.  With rows laid out by label most rows of the pair find their
// minimum next to it, so every role visits its tile first (tiles in rotated
// order) and the epilogue visits its 32-column chunk first within that tile:
// the running minimum is set at once and the other chunks are skipped.
// Visiting order never changes results (certified rows have one candidate;
// ambiguous rows are resolved exactly, lowest index on ties).
__device__ __forceinline__ int sb_first_col(const int32_t* lprev, const int32_t* orig, int64_t pr, int64_t n, int k,
                                            int rows) {
  if (lprev == nullptr) return 0;
  int64_t r = pr * rows + rows / 2;
  if (r >= n) r = pr * rows;
  const int l = lprev[orig != nullptr ? (int64_t)orig[r] : r];
  return (l >= 0 && l < k) ? l : 0;
}

// Rows handled by a launch: pass 1 = n; pass 2 = the device-side ambiguous
// count, or 0 when the resolver is bypassed (count above `bypass`).
__device__ __forceinline__ int64_t sb_rows(int64_t n, const int* amb_count, int64_t bypass) {
  if (amb_count == nullptr) return n;
  const int64_t c = *(volatile const int*)amb_count;
  return c > bypass ? 0 : c;
}

// Minimum of a 32-key chunk: a depth-4 tree of 3-input mins (16 FMNMX3).
__device__ __forceinline__ float sb_chunk_min(const uint32_t (&c)[32]) {
  float t[11];
#pragma unroll
  for (int i = 0; i < 10; ++i)
    t[i] = fmin3(__uint_as_float(c[3 * i]), __uint_as_float(c[3 * i + 1]), __uint_as_float(c[3 * i + 2]));
  t[10] = fminf(__uint_as_float(c[30]), __uint_as_float(c[31]));
  return fminf(fmin3(fmin3(t[0], t[1], t[2]), fmin3(t[3], t[4], t[5]), fmin3(t[6], t[7], t[8])), fminf(t[9], t[10]));
}

// Pass 2 (candidate emission) on one 32-key chunk (columns col ..): the
// candidate mask (FSETP + SEL per key), then a short loop over its set bits
// (2-3 candidates per row in total).
__device__ __forceinline__ void sb_chunk_cand(const uint32_t (&cur)[32], int col, float thr, int64_t row, int64_t n,
                                              int64_t rc, int* __restrict__ cand, int& nc) {
  uint32_t bits = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) bits |= (__uint_as_float(cur[i]) <= thr ? 1u : 0u) << i;
  while (bits) {
    const int i = __ffs(bits) - 1;
    bits &= bits - 1;
    if (row < n && nc < SB_NCAND) cand[rc * SB_NCAND + nc] = col + i;
    ++nc;
  }
}

// Full update of one chunk (running best two packed keys, exact count).
__device__ __forceinline__ void sb_chunk_full(const uint32_t (&cur)[32], int col, float twoE, uint32_t msk,
                                              float& R1, int& r1, float& R2, int& r2, float& cnt) {
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(cur[i]);
  screen_chunk_top2(v, msk, col, twoE, R1, r1, R2, r2, cnt);
}

// Chunk skip threshold of the running minimum: a chunk whose smallest key is
// above it for every row of the warp leaves (R1, r1, R2, r2, cnt) unchanged.
__device__ __forceinline__ float sb_skip_thr(float R1, float twoE) {
  return (R1 + twoE + 0x1p-16f * fabsf(R1)) * (1.0f + 0x1p-16f);
}

template <int NKC, bool CAND, bool W, bool F8, int RT, int CB>
__global__ void __launch_bounds__(SB_THREADS, 1)
assign_screen_bf16_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                          const __grid_constant__ CUtensorMap tm_baug, const float* __restrict__ anorm,
                          const float* __restrict__ danorm, const float* __restrict__ bstat, int64_t n_in, int k,
                          int32_t* __restrict__ labels, int* __restrict__ amb_list, int* __restrict__ amb_count,
                          float* __restrict__ amb_thr, int64_t bypass, int* __restrict__ cand,
                          int* __restrict__ cand_n, const int32_t* __restrict__ orig,
                          const int32_t* __restrict__ lprev, int* __restrict__ two_list, int* __restrict__ two_count,
                          const long long* __restrict__ state) {
  using Cfg = SbCfg<NKC, W, RT, CB>;
  constexpr int BN = Cfg::kBN, CH = Cfg::kChunks, STAGES = Cfg::kStages, PR = Cfg::kRows;
  constexpr int XC = CB / 2;  // chunk width in the tensor maps' BF16 units
  auto sdesc = [](uint32_t a) { return CB == 128 ? ptx::sdesc_k_sw128(a) : ptx::sdesc_k_sw64(a); };
  if (stopped(state)) return;
  const int64_t n = CAND ? sb_rows(n_in, amb_count, bypass) : n_in;
  if (n == 0) return;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + Cfg::kABytes;
  uint8_t* sAaug = sB + STAGES * Cfg::kStageB;
  uint8_t* bar_area = sAaug + Cfg::kAAug;
  constexpr int AS = Cfg::kAStages;
  uint64_t* afull = reinterpret_cast<uint64_t*>(bar_area);  // [AS][NKC]
  uint64_t* aempty = afull + AS * NKC;                       // [AS][NKC]
  uint64_t* full = aempty + AS * NKC;                        // [STAGES]
  uint64_t* empty = full + STAGES;                           // [STAGES]
  uint64_t* tfull = empty + STAGES;                          // [2 buffers][2 row tiles] (W: [row tile])
  uint64_t* tempty = tfull + 4;                              // [2][2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 4);

  // warp index through a shuffle: provably warp-uniform, so role branches and the
  // MMA loop's bookkeeping stay in uniform registers
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int ntiles = (k + BN - 1) / BN;
  const float OFF = bstat[2];
  // constant A columns of the augmented K step, no-swizzle K-major layout
  // [2 K halves][128 rows][16 B]: every row = (1, 1, 1, 0, ..., 0), so the MMA
  // adds h1 + h2 + h3 = |c|^2 + OFF (the B side) to -2 <p~, c~>: the paper's
  // augmented form q.C.q^T with q = [p, 1] computed by the tensor core.
  for (int i = threadIdx.x; i < 2 * 128; i += blockDim.x) {
    const uint32_t one2 = 0x3F803F80u;  // bf16 (1, 1)
    uint4 u = make_uint4(0u, 0u, 0u, 0u);
    if (i < 128) u = make_uint4(one2, 0x00003F80u, 0u, 0u);
    reinterpret_cast<uint4*>(sAaug)[i] = u;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic stores -> UMMA reads
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tm_a);
    ptx::prefetch_tmap(&tm_b);
    ptx::prefetch_tmap(&tm_baug);
    for (int c = 0; c < NKC; ++c) {
      for (int a = 0; a < AS; ++a) {
        ptx::mbar_init(&afull[a * NKC + c], 1);
        ptx::mbar_init(&aempty[a * NKC + c], 1);
      }
    }
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 4; ++b) {  // one row tile's accumulator each: its 4 epilogue warps release it
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], 128);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t npairs = (n + PR - 1) / PR;
  // registers: the producer / MMA warpgroup needs few, the two epilogue
  // warpgroups hold two chunk pairs of keys (128 registers) in flight
  if (warp < 4) {
  ptx::regs_dec<SbCfg<NKC, W, RT, CB>::kRegsLow>();
  if (warp == 0) {
    // ---------------- A producer: both row tiles, chunk by chunk ----------------
    const uint64_t pol = ptx::policy_evict_first();
    int it = 0;
    for (int64_t pr = blockIdx.x; pr < npairs; pr += gridDim.x, ++it) {
      for (int c = 0; c < NKC; ++c) {
        const int ab = it % AS;
        uint8_t* sAp = sA + ab * Cfg::kAPair;
        if (it >= AS) ptx::mbar_wait(&aempty[ab * NKC + c], (uint32_t)((it / AS - 1) & 1));
        if (ptx::elect_one()) {
          ptx::mbar_expect_tx(&afull[ab * NKC + c], RT * Cfg::kTileBytes);
          ptx::tma_load_2d(&tm_a, &afull[ab * NKC + c], sAp + (0 * NKC + c) * Cfg::kTileBytes, c * XC,
                           (int)(pr * PR), pol);
          if (RT == 2)
            ptx::tma_load_2d(&tm_a, &afull[ab * NKC + c], sAp + (1 * NKC + c) * Cfg::kTileBytes, c * XC,
                             (int)(pr * PR + 128), pol);
        }
        __syncwarp();
      }
    }
  } else if (warp == 3) {
    // ---------------- B producer: centroid chunks through the ring ----------------
    const uint64_t pol = ptx::policy_evict_last();
    int stage = 0;
    uint32_t phase = 0;
    // first tile of the next pair fetched one pair ahead (two dependent
    // global loads would otherwise stall the ring at every pair boundary)
    int t0_nx = blockIdx.x < npairs ? sb_first_col(lprev, orig, blockIdx.x, n, k, PR) / BN : 0;
    for (int64_t pr = blockIdx.x; pr < npairs; pr += gridDim.x) {
      const int t0 = t0_nx;
      if (pr + gridDim.x < npairs) t0_nx = sb_first_col(lprev, orig, pr + gridDim.x, n, k, PR) / BN;
      for (int nt = 0; nt < ntiles; ++nt) {
        const int tile = nt + t0 < ntiles ? nt + t0 : nt + t0 - ntiles;
        for (int c = 0; c < NKC; ++c) {
          ptx::mbar_wait(&empty[stage], phase ^ 1u);
          if (ptx::elect_one()) {
            uint8_t* st = sB + stage * Cfg::kStageB;
            const bool last = c + 1 == NKC;  // the tile's augmented columns ride with its last chunk
            {
            ptx::mbar_expect_tx(&full[stage], Cfg::kBBytes + (last ? Cfg::kAugBytes : 0u));
            ptx::tma_load_2d(&tm_b, &full[stage], st, c * XC, tile * BN, pol);
            if (last) {
              ptx::tma_load_2d(&tm_baug, &full[stage], st + Cfg::kBBytes, 0, tile * BN, pol);
              ptx::tma_load_2d(&tm_baug, &full[stage], st + Cfg::kBBytes + BN * 16, 8, tile * BN, pol);
            }
            }
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (warp-uniform loop, one elected lane issues) ----------------
    constexpr uint32_t idesc = ptx::idesc_bf16<128, BN>();  // the augmented K step is BF16 in both modes
    constexpr uint32_t idesc_main = F8 ? ptx::idesc_e4m3<128, BN>() : idesc;
    // main K steps: 32 bytes of each operand row per MMA (K = 16 BF16 / 32 E4M3)
    auto mma_main = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
      if constexpr (F8) ptx::umma_f8(d, a, b, idesc_main, acc);
      else ptx::umma_f16(d, a, b, idesc_main, acc);
    };
    if constexpr (W) {
      // both row tiles per centroid tile; the tile's NKC chunk stages stay
      // resident until the second row tile's MMAs have read them
      int stage = 0;
      uint32_t phase = 0, tpar = 0;
      int it = 0;
      for (int64_t pr = blockIdx.x; pr < npairs; pr += gridDim.x, ++it) {
        for (int nt = 0; nt < ntiles; ++nt) {
          int stc[NKC];
          uint32_t phc[NKC];
#pragma unroll
          for (int c = 0; c < NKC; ++c) {
            stc[c] = stage;
            phc[c] = phase;
            if (++stage == STAGES) { stage = 0; phase ^= 1u; }
          }
#pragma unroll
          for (int rt = 0; rt < 2; ++rt) {
            ptx::mbar_wait(&tempty[rt], tpar ^ 1u);
            ptx::tc_fence_after();
            const uint32_t d0 = tmem + (uint32_t)(rt * 256);
#pragma unroll
            for (int c = 0; c < NKC; ++c) {
              if (rt == 0) {
                if (nt == 0) ptx::mbar_wait(&afull[c], (uint32_t)(it & 1));
                ptx::mbar_wait(&full[stc[c]], phc[c]);
                ptx::tc_fence_after();
              }
              const uint64_t ad = sdesc(ptx::smem_u32(sA + (rt * NKC + c) * Cfg::kTileBytes));
              const uint64_t bd = sdesc(ptx::smem_u32(sB + stc[c] * Cfg::kStageB));
              if (ptx::elect_one()) {
#pragma unroll
                for (int ks = 0; ks < Cfg::kKSteps; ++ks) {
                  const uint64_t off = (uint64_t)(ks * 32) >> 4;
                  mma_main(d0, ad + off, bd + off, (c | ks) != 0);
                }
                if (c + 1 == NKC) {
                  const uint64_t aa = ptx::sdesc_k_none(ptx::smem_u32(sAaug), 128 * 16, 128);
                  const uint64_t ba = ptx::sdesc_k_none(ptx::smem_u32(sB + stc[c] * Cfg::kStageB + Cfg::kBBytes),
                                                        BN * 16, 128);
                  ptx::umma_f16(d0, aa, ba, idesc, 1u);
                }
              }
              __syncwarp();
            }
            if (ptx::elect_one()) ptx::umma_commit(&tfull[rt]);
            __syncwarp();
          }
          if (ptx::elect_one()) {
#pragma unroll
            for (int c = 0; c < NKC; ++c) {
              ptx::umma_commit(&empty[stc[c]]);
              if (nt + 1 == ntiles) ptx::umma_commit(&aempty[c]);
            }
          }
          __syncwarp();
          tpar ^= 1u;
        }
      }
    } else {
    int stage = 0;
    uint32_t phase = 0;
    int abuf = 0;
    uint32_t aphase = 0;
    int it = 0;
    // Per centroid tile: all K steps of row tile 0, handed to its 4 epilogue
    // warps, then row tile 1 — each row tile's accumulator is released by its
    // own warps, and row tile 0's epilogue starts while row tile 1's MMAs run.
    for (int64_t pr = blockIdx.x; pr < npairs; pr += gridDim.x, ++it) {
      const int ab = it % AS;
      uint8_t* sAp = sA + ab * Cfg::kAPair;
      for (int nt = 0; nt < ntiles; ++nt) {
        int stc[NKC];
        uint32_t phc[NKC];
#pragma unroll
        for (int c = 0; c < NKC; ++c) {
          stc[c] = stage;
          phc[c] = phase;
          if (++stage == STAGES) { stage = 0; phase ^= 1u; }
        }
#pragma unroll
        for (int rt = 0; rt < RT; ++rt) {
          ptx::mbar_wait(&tempty[abuf * 2 + rt], aphase ^ 1u);
          ptx::tc_fence_after();
          const uint32_t d0 = tmem + (uint32_t)(abuf * 256 + rt * 128);
#pragma unroll
          for (int c = 0; c < NKC; ++c) {
            if (rt == 0) {
              if (nt == 0) ptx::mbar_wait(&afull[ab * NKC + c], (uint32_t)((it / AS) & 1));
              ptx::mbar_wait(&full[stc[c]], phc[c]);
              ptx::tc_fence_after();
            }
            const uint64_t a0 = sdesc(ptx::smem_u32(sAp + (rt * NKC + c) * Cfg::kTileBytes));
            const uint64_t bd = sdesc(ptx::smem_u32(sB + stc[c] * Cfg::kStageB));
            if (ptx::elect_one()) {
#pragma unroll
              for (int ks = 0; ks < Cfg::kKSteps; ++ks) {  // 32 bytes of each row per MMA
                const uint64_t off = (uint64_t)(ks * 32) >> 4;
                mma_main(d0, a0 + off, bd + off, (c | ks) != 0);
              }
              if (c + 1 == NKC) {  // augmented K step: + (|c|^2 + OFF) in three BF16 pieces
                const uint64_t aa = ptx::sdesc_k_none(ptx::smem_u32(sAaug), 128 * 16, 128);
                const uint64_t ba = ptx::sdesc_k_none(ptx::smem_u32(sB + stc[c] * Cfg::kStageB + Cfg::kBBytes),
                                                      BN * 16, 128);
                ptx::umma_f16(d0, aa, ba, idesc, 1u);
              }
              if (rt + 1 == RT) {
                ptx::umma_commit(&empty[stc[c]]);
                if (nt + 1 == ntiles) ptx::umma_commit(&aempty[ab * NKC + c]);  // A chunk free again
              }
            }
            __syncwarp();
          }
          if (ptx::elect_one()) ptx::umma_commit(&tfull[abuf * 2 + rt]);
          __syncwarp();
        }
        abuf ^= 1;
        if (abuf == 0) aphase ^= 1u;
      }
    }
    }  // !W
  }
  } else {
  ptx::regs_inc<SbCfg<NKC, W, RT, CB>::kRegsHigh>();
  if (warp < 4 + 4 * RT) {
    // ---------------- epilogue: warp (g, h) = lanes 32g.. of row tile h ----------------
    const int g = warp & 3, h = (warp - 4) >> 2;
    const float Bmax = bstat[0], dBmax = bstat[1];
    // BF16 / E4M3 products are exact in f32; each MMA adds at most (K + 1)
    // roundings relative to the running sum of |products| (K = 16 / 32)
    const float acc_rel = (float)(NKC * 4 + 3) * (F8 ? 0x1p-18f : 0x1p-19f);
    const float kscale = bstat[4];  // keys come out of the MMA scaled by S = sp * sc (1 for BF16)
    const uint32_t msk = kIdxMask;
    int abuf = 0;
    uint32_t aphase = 0;
    const int64_t r_in = h * 128 + g * 32 + lane;
    // TMEM of this warp's 32 rows: W = its row tile's single 256-column
    // accumulator; otherwise buffer b at columns b * 256 + h * 128
    const uint32_t tlane = tmem + ((uint32_t)(g * 32) << 16) + (uint32_t)(h * (W ? 256 : 128));
    uint32_t tph = 0;  // W: phase of this row tile's accumulator
    auto tbar = [&]() { return W ? h : abuf * 2 + h; };
    auto tphase = [&]() { return W ? tph : aphase; };
    auto tbase = [&]() { return tlane + (uint32_t)(W ? 0 : abuf * 256); };
    auto tnext = [&]() {
      if (W) {
        tph ^= 1u;
      } else {
        abuf ^= 1;
        if (abuf == 0) aphase ^= 1u;
      }
    };
    // N = 128 tiles (X4 below): a tile's four 32-column chunks are loaded at
    // once into (vA0, vA1, vB0, vB1) and the accumulator is handed back after a
    // single tcgen05.wait::ld, before any arithmetic — the MMAs wait on this
    // release (two accumulators per row tile), not on the arithmetic.
    // N = 256 tiles (W): loads run one chunk PAIR ahead of the arithmetic, two
    // loads per wait, buffers (vA0, vA1) / (vB0, vB1) alternating by pair
    // parity across tile and pair boundaries.  The epilogue warpgroups run at
    // 200 registers (setmaxnreg).
    constexpr int CP = CH / 2;
    static_assert(CH % 4 == 0, "chunk pairs alternate buffers across tiles");
    uint32_t vA0[32], vA1[32], vB0[32], vB1[32];
    // per-row inputs of the next pair are fetched one pair ahead: their DRAM
    // latency would otherwise hold both TMEM buffers (and the MMAs) at every
    // pair boundary
    // Loaded values are kept raw (32-bit) until used: a conversion right after
    // the load (e.g. sign-extending a row id) would wait for it at once.  The
    // first column (orig -> previous label) is a dependent pair of loads: the
    // second one is issued a chunk later (fetch_pair_b).
    float an_nx = 0.0f, dan_nx = 0.0f;
    unsigned fc_nx = 0;  // first column of the next pair (unsigned: / and % are shifts)
    int out_nx = 0, mid_nx = 0;
    auto fetch_pair = [&](int64_t p) {
      const int64_t rr = p * PR + r_in < n ? p * PR + r_in : n - 1;
      out_nx = (!CAND && orig != nullptr) ? orig[rr] : (int)rr;
      if (CAND) {
        an_nx = amb_thr[rr];
      } else {
        an_nx = anorm[rr];
        dan_nx = danorm[rr];
      }
      int64_t rm = p * PR + PR / 2;
      if (rm >= n) rm = p * PR;
      mid_nx = (lprev != nullptr && orig != nullptr) ? orig[rm] : (int)rm;
    };
    auto fetch_pair_b = [&]() {
      const int l = lprev != nullptr ? lprev[mid_nx] : 0;
      fc_nx = (l >= 0 && l < k) ? (unsigned)l : 0u;
    };
    // X4: no loads run ahead across tiles.  Measured against the pair-ahead
    // scheme (PCB_EPI_X4=0): c3 1.232 vs 1.290 ms, c5 38.1 vs 37.8 ms
    constexpr bool X4 = PCB_EPI_X4 && !W && CH == 4;
    if (X4 && blockIdx.x < npairs) {
      fetch_pair(blockIdx.x);
      fetch_pair_b();
    } else if (blockIdx.x < npairs) {
      fetch_pair(blockIdx.x);
      fetch_pair_b();
      ptx::mbar_wait(&tfull[tbar()], 0);
      ptx::tc_fence_after();
      const int q0 = (int)((fc_nx % BN) / 32);
      ptx::tmem_ld_32x32b_x32_async(tbase() + 32 * q0, vA0);
      ptx::tmem_ld_32x32b_x32_async(tbase() + 32 * ((q0 + 1) & (CH - 1)), vA1);
    }
    for (int64_t pr = blockIdx.x; pr < npairs; pr += gridDim.x) {
      const int64_t row = pr * PR + r_in;
      const int64_t rc = row < n ? row : n - 1;
      const bool last_pair = pr + gridDim.x >= npairs;
      float twoE = 0.0f, big = 0.0f, thr = 0.0f;
      int nc = 0;
      if (CAND) {
        thr = an_nx;
      } else {
        twoE = kscale * screen_two_e_aug(an_nx, dan_nx, Bmax, dBmax, OFF, acc_rel);
        big = 64.0f / twoE;
      }
      (void)big;
      const int t0 = (int)(fc_nx / BN), q0 = (int)((fc_nx % BN) / 32);
      const int out_row = out_nx;  // original row id (label store)
      if (!last_pair) fetch_pair(pr + gridDim.x);
      float R1 = 3.4e38f, R2 = 3.4e38f, cnt = 0.0f;
      int r1 = 0, r2 = 0;
      float thr_skip = 3.4e38f;  // sb_skip_thr(R1, twoE), refreshed when R1 changes
      auto pair_work = [&](const uint32_t (&cur0)[32], const uint32_t (&cur1)[32], int ca, int cb) {
        if (CAND) {
          sb_chunk_cand(cur0, ca, thr, row, n, rc, cand, nc);
          sb_chunk_cand(cur1, cb, thr, row, n, rc, cand, nc);
        } else {
          const float m0 = sb_chunk_min(cur0), m1 = sb_chunk_min(cur1);
          if (__any_sync(0xffffffffu, fminf(m0, m1) <= thr_skip)) {
            if (__any_sync(0xffffffffu, m0 <= thr_skip)) sb_chunk_full(cur0, ca, twoE, msk, R1, r1, R2, r2, cnt);
            if (__any_sync(0xffffffffu, m1 <= sb_skip_thr(R1, twoE)))
              sb_chunk_full(cur1, cb, twoE, msk, R1, r1, R2, r2, cnt);
            thr_skip = sb_skip_thr(R1, twoE);
          }
        }
      };
      if constexpr (X4) {
        for (int nt = 0; nt < ntiles; ++nt) {
          const int c0 = (nt + t0 < ntiles ? nt + t0 : nt + t0 - ntiles) * BN;
          const int qr = nt == 0 ? q0 : 0;  // the first tile starts at the previous label's chunk
          ptx::mbar_wait(&tfull[tbar()], tphase());
          ptx::tc_fence_after();
          const uint32_t taddr = tbase();
          ptx::tmem_ld_32x32b_x32_async(taddr + 32 * qr, vA0);
          ptx::tmem_ld_32x32b_x32_async(taddr + 32 * ((qr + 1) & 3), vA1);
          ptx::tmem_ld_32x32b_x32_async(taddr + 32 * ((qr + 2) & 3), vB0);
          ptx::tmem_ld_32x32b_x32_async(taddr + 32 * ((qr + 3) & 3), vB1);
          ptx::tmem_wait_ld(vA0);
          ptx::tie_regs(vA1);
          ptx::tie_regs(vB0);
          ptx::tie_regs(vB1);
          ptx::tc_fence_before();
          ptx::mbar_arrive(&tempty[tbar()]);
          tnext();
          if (nt == 0 && !last_pair) fetch_pair_b();
          pair_work(vA0, vA1, c0 + 32 * qr, c0 + 32 * ((qr + 1) & 3));
          pair_work(vB0, vB1, c0 + 32 * ((qr + 2) & 3), c0 + 32 * ((qr + 3) & 3));
        }
      } else
      for (int nt = 0; nt < ntiles; ++nt) {
        const uint32_t taddr = tbase();
        const int c0 = (nt + t0 < ntiles ? nt + t0 : nt + t0 - ntiles) * BN;
#pragma unroll
        for (int p = 0; p < CP; ++p) {
          uint32_t (&cur0)[32] = (p & 1) ? vB0 : vA0;
          uint32_t (&cur1)[32] = (p & 1) ? vB1 : vA1;
          uint32_t (&nxt0)[32] = (p & 1) ? vA0 : vB0;
          uint32_t (&nxt1)[32] = (p & 1) ? vA1 : vB1;
          ptx::tmem_wait_ld(cur0);
          ptx::tie_regs(cur1);
          if (nt == 0 && p == CP - 1 && !last_pair) fetch_pair_b();  // its first load was issued a tile ago
          // chunks of the tile held by cur0 / cur1 (the first tile starts at the previous label's chunk)
          const int qa = nt == 0 ? ((2 * p + q0) & (CH - 1)) : 2 * p;
          const int qb = nt == 0 ? ((2 * p + 1 + q0) & (CH - 1)) : 2 * p + 1;
          if (p < CP - 1) {
            const int qn = nt == 0 ? ((2 * p + 2 + q0) & (CH - 1)) : 2 * p + 2;
            const int qm = nt == 0 ? ((2 * p + 3 + q0) & (CH - 1)) : 2 * p + 3;
            ptx::tmem_ld_32x32b_x32_async(taddr + 32 * qn, nxt0);
            ptx::tmem_ld_32x32b_x32_async(taddr + 32 * qm, nxt1);
          } else {
            // this accumulator is fully read: hand it back, prefetch the next one
            ptx::tc_fence_before();
            ptx::mbar_arrive(&tempty[tbar()]);
            tnext();
            if (nt + 1 < ntiles || !last_pair) {
              ptx::mbar_wait(&tfull[tbar()], tphase());
              ptx::tc_fence_after();
              // first chunks of the next pair: read fc_nx only here, a pair after
              // its (two dependent) loads were issued
              const int qn = nt + 1 < ntiles ? 0 : (int)((fc_nx % BN) / 32);
              ptx::tmem_ld_32x32b_x32_async(tbase() + 32 * qn, nxt0);
              ptx::tmem_ld_32x32b_x32_async(tbase() + 32 * ((qn + 1) & (CH - 1)), nxt1);
            }
          }
          // chunk skip, decided per pair: rows are laid out by label
          // (pcb_screen_relayout_bf16), so the rows of a warp see their
          // minima in the same chunks and most pairs of most warps skip
          pair_work(cur0, cur1, c0 + 32 * qa, c0 + 32 * qb);
        }
      }
      if (CAND) {
        if (row < n) cand_n[row] = nc;
      } else {
        if (row < n) labels[out_row] = r1;
        // exactly two keys within the bound: the candidates are r1, r2 (exact
        // f64 resolution, no second pass); more: pass 2 finds them
        const bool two = row < n && cnt == 2.0f;
        const unsigned m2 = __ballot_sync(0xffffffffu, two);
        if (m2) {
          int base = 0;
          if (lane == 0) base = atomicAdd(two_count, __popc(m2));
          base = __shfl_sync(0xffffffffu, base, 0);
          if (two) {
            const int pos = base + __popc(m2 & ((1u << lane) - 1u));
            two_list[3 * pos + 0] = (int)out_row;
            two_list[3 * pos + 1] = r1;
            two_list[3 * pos + 2] = r2;
          }
        }
        const bool amb = row < n && cnt > 2.0f;
        const unsigned m = __ballot_sync(0xffffffffu, amb);
        if (m) {
          int base = 0;
          if (lane == 0) base = atomicAdd(amb_count, __popc(m));
          base = __shfl_sync(0xffffffffu, base, 0);
          if (amb) {
            const int pos = base + __popc(m & ((1u << lane) - 1u));
            amb_list[pos] = (int)row;
            // R1 carries a 5-bit index in its low mantissa bits: 2^-17 relative slack
            amb_thr[pos] = (R1 + twoE) * (1.0f + 0x1p-14f);
          }
        }
      }
    }
  }
  }  // epilogue warpgroups
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc<512>(tmem);
}

static int make_tmap_bf16(CUtensorMap* m, const __nv_bfloat16* base, int64_t rows, int cols, int box_rows,
                          int box_cols = SB_BKE, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
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
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<__nv_bfloat16*>(base), dims, strides, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : PCB_EINVAL;
}

template <int NKC, bool CAND, bool W, bool F8, int RT = 2, int CB = 128>
static int launch_screen_bf16(const __nv_bfloat16* A, int64_t n, const __nv_bfloat16* B, int k,
                              const float* an, const float* dan, const __nv_bfloat16* Baug, const float* bstat,
                              int32_t* labels, int* amb_list, int* amb_count, float* amb_thr, int64_t bypass,
                              int* cand, int* cand_n, const int32_t* orig, const int32_t* lprev,
                              int* two_list, int* two_count, const long long* state, cudaStream_t st) {
  using Cfg = SbCfg<NKC, W, RT, CB>;
  CUtensorMap ta, tb, tg;
  int rc;
  const int64_t kpad = (k + SB_KPAD - 1) / SB_KPAD * SB_KPAD;  // B / Baug hold kpad rows (padding: key = +huge)
  // CB-byte chunks (E4M3 rows viewed as BF16 pairs)
  const CUtensorMapSwizzle swz = CB == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  if ((rc = make_tmap_bf16(&ta, A, n, NKC * CB / 2, 128, CB / 2, swz))) return rc;
  if ((rc = make_tmap_bf16(&tb, B, kpad, NKC * CB / 2, Cfg::kBN, CB / 2, swz))) return rc;
  if ((rc = make_tmap_bf16(&tg, Baug, kpad, SB_AUG, Cfg::kBN, 8, CU_TENSOR_MAP_SWIZZLE_NONE))) return rc;
  auto kern = assign_screen_bf16_kernel<NKC, CAND, W, F8, RT, CB>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::kSmem);
  if (e != cudaSuccess) return (int)e;
  {
    // the setmaxnreg split assumes the launch allocation ptxas was given
    static int regs = -1;
    if (regs < 0) {
      cudaFuncAttributes fa;
      if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess) return PCB_ENODEV;
      regs = fa.numRegs;
    }
    if (regs != Cfg::kLaunchRegs) return PCB_EUNSUP;
  }
  const int64_t npairs = (n + Cfg::kRows - 1) / Cfg::kRows;
  const int grid = (int)std::min<int64_t>(npairs, (int64_t)sm_count());
  kern<<<grid, SB_THREADS, Cfg::kSmem, st>>>(ta, tb, tg, an, dan, bstat, n, k, labels, amb_list, amb_count,
                                             amb_thr, bypass, cand, cand_n, orig, lprev, two_list, two_count, state);
  PCB_CHECK_LAUNCH();
  return 0;
}

template <bool CAND, bool F8 = false>
static int dispatch_bf16(int ldb, const __nv_bfloat16* A, int64_t n, const __nv_bfloat16* B, int k,
                         const float* an, const float* dan, const __nv_bfloat16* Baug, const float* bstat,
                         int32_t* labels, int* amb_list, int* amb_count, float* amb_thr, int64_t bypass,
                         int* cand, int* cand_n, const int32_t* orig, const int32_t* lprev, int* two_list,
                         int* two_count, const long long* state, cudaStream_t st) {
#define PCB_SB_CASE(N, WIDE)                                                                                \
    return launch_screen_bf16<N, CAND, WIDE, F8>(A, n, B, k, an, dan, Baug, bstat, labels, amb_list, amb_count, \
                                             amb_thr, bypass, cand, cand_n, orig, lprev, two_list, two_count, \
                                             state, st);
  // d <= 128: N = 128 tiles; PCB_SCREEN_WIDE=1 selects the N = 256 layout
  // (measured slower at c3 / c5: 2.52 vs 2.37 ms, 65 vs 56 ms; MMA-only 2.14
  // vs 2.03 ms — the BF16 MMA rate, not shared-memory operand bandwidth, binds)
  static const bool narrow = getenv("PCB_SCREEN_WIDE") == nullptr;
  if (F8 && ldb == 32)  // E4M3 rows of 64 bytes (d <= 64): SWIZZLE_64B chunks
    return launch_screen_bf16<1, CAND, false, F8, 2, 64>(A, n, B, k, an, dan, Baug, bstat, labels, amb_list,
                                                        amb_count, amb_thr, bypass, cand, cand_n, orig, lprev,
                                                        two_list, two_count, state, st);
  switch (ldb / SB_BKE) {
    case 1: if (narrow) { PCB_SB_CASE(1, false) } else { PCB_SB_CASE(1, true) }
    case 2: if (narrow) { PCB_SB_CASE(2, false) } else { PCB_SB_CASE(2, true) }
    case 3: PCB_SB_CASE(3, false)
    case 4: PCB_SB_CASE(4, false)
#define PCB_SB_CASE1(N)                                                                                     \
    return launch_screen_bf16<N, CAND, false, F8, 1>(A, n, B, k, an, dan, Baug, bstat, labels, amb_list,    \
                                                     amb_count, amb_thr, bypass, cand, cand_n, orig, lprev,  \
                                                     two_list, two_count, state, st);
    // longer rows: one resident row tile of 128 (the operand chunks of two would not fit)
    case 5: PCB_SB_CASE1(5)
    case 6: PCB_SB_CASE1(6)
    case 7: PCB_SB_CASE1(7)
    case 8: PCB_SB_CASE1(8)
#undef PCB_SB_CASE1
    default: return PCB_EUNSUP;
  }
#undef PCB_SB_CASE
}

// ---- prep: RN BF16 copies and the residual norms of the bound ----------------------

__device__ __forceinline__ void atomic_max_pos_f(float* addr, float v) {
  atomicMax(reinterpret_cast<unsigned int*>(addr), __float_as_uint(v));  // v >= 0
}

// Per row of X (rows x d): |bf16(x)|, |x - bf16(x)| (rounded up), max |x|^2 and
// the BF16 copy Xb (row stride ldb, zero padded).
__global__ void __launch_bounds__(256)
row_bf16_norms_kernel(const float* __restrict__ X, int64_t rows, int d, float* __restrict__ an,
                      float* __restrict__ dan, float* __restrict__ maxsq, __nv_bfloat16* __restrict__ Xb, int ldb,
                      float out_scale = 1.0f) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float wmax = 0.0f;
  for (int64_t i = w; i < rows; i += nw) {
    double s_t = 0.0, s_d = 0.0, s_x = 0.0;
    for (int t = lane; t < ldb; t += 32) {
      const float x = t < d ? X[i * d + t] : 0.0f;
      const __nv_bfloat16 hb = __float2bfloat16_rn(x);
      Xb[i * ldb + t] = out_scale == 1.0f ? hb : __float2bfloat16_rn(out_scale * __bfloat162float(hb));  // exact
      const double h = (double)__bfloat162float(hb);
      const double dd = (double)x - h;
      s_t = fma(h, h, s_t);
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
  if (lane == 0 && maxsq != nullptr) atomic_max_pos_f(maxsq, wmax);
}

__global__ void max2_bf16_kernel(const float* __restrict__ b, const float* __restrict__ db, int k,
                                 float* __restrict__ out) {
  float m0 = 0.0f, m1 = 0.0f;
  for (int j = threadIdx.x; j < k; j += blockDim.x) { m0 = fmaxf(m0, b[j]); m1 = fmaxf(m1, db[j]); }
  atomic_max_pos_f(&out[0], m0);
  atomic_max_pos_f(&out[1], m1);
}

__global__ void screen_off_kernel(float* __restrict__ bstat, const float* __restrict__ maxsq) {
  bstat[4] = 1.0f;  // key scale (BF16: the MMA emits unscaled keys)
  bstat[2] = 1.01f * (*maxsq) + 1.0f;  // OFF > max |p|^2: every key positive
}

// Compact copy of the ambiguous rows of Xb (pass-2 input).
__global__ void __launch_bounds__(256)
gather_rows_bf16(const __nv_bfloat16* __restrict__ Xb, int ldb, const int* __restrict__ list,
                 const int* __restrict__ count, int64_t bypass, __nv_bfloat16* __restrict__ out,
                 const long long* __restrict__ state) {
  if (stopped(state)) return;
  const int64_t cnt = *count;
  if (cnt > bypass) return;
  const int per = ldb / 8;  // 16-byte vectors per row
  const int64_t total = cnt * per;
  const uint4* src = reinterpret_cast<const uint4*>(Xb);
  uint4* dst = reinterpret_cast<uint4*>(out);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / per, q = e - r * per;
    dst[r * per + q] = src[(int64_t)list[r] * per + q];
  }
}

// Four consecutive floats q*4 .. q*4+3 of a row (zero past d); 16-byte load
// when the row is 16-byte aligned (d % 4 == 0).
__device__ __forceinline__ float4 load4(const float* __restrict__ rowp, int q, int d) {
  const int t = 4 * q;
  if ((d & 3) == 0) return t < d ? __ldg(reinterpret_cast<const float4*>(rowp) + q) : make_float4(0, 0, 0, 0);
  return make_float4(t < d ? rowp[t] : 0.0f, t + 1 < d ? rowp[t + 1] : 0.0f, t + 2 < d ? rowp[t + 2] : 0.0f,
                     t + 3 < d ? rowp[t + 3] : 0.0f);
}
__device__ __forceinline__ float dist4f(float4 a, float4 b, float s) {
  const float e0 = a.x - b.x, e1 = a.y - b.y, e2 = a.z - b.z, e3 = a.w - b.w;
  return fmaf(e3, e3, fmaf(e2, e2, fmaf(e1, e1, fmaf(e0, e0, s))));
}
__device__ __forceinline__ double dist4(float4 a, float4 b, double s) {
  const double e0 = (double)a.x - (double)b.x, e1 = (double)a.y - (double)b.y;
  const double e2 = (double)a.z - (double)b.z, e3 = (double)a.w - (double)b.w;
  return fma(e3, e3, fma(e2, e2, fma(e1, e1, fma(e0, e0, s))));
}

// Rows longer than 256: 8 lanes per ambiguous row (4 rows per warp, float4
// lanes, 4 loads of each row in flight), f32 distances with the (d + 8) 2^-23
// margin, f64 for thin margins; same lists, ties to the lowest index.
__global__ void __launch_bounds__(256, 3)
screen_exact_wide_kernel(const float* __restrict__ P, int d, const float* __restrict__ C,
                         const int* __restrict__ list, const int* __restrict__ count, int64_t bypass,
                         const int* __restrict__ cand, const int* __restrict__ cand_n, int32_t* __restrict__ labels,
                         int* __restrict__ ovf_list, int* __restrict__ ovf_count, const int32_t* __restrict__ orig,
                         const int* __restrict__ two_list, const int* __restrict__ two_count,
                         const long long* __restrict__ state) {
  if (stopped(state)) return;
  const int64_t cnt_amb = *count;
  const int64_t cnt2 = two_count != nullptr ? *two_count : 0;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool bypassed = cnt_amb > bypass;
  if (bypassed) {
    for (int64_t b0 = w0 * 32; b0 < cnt_amb; b0 += nw * 32) {
      const int64_t r = b0 + lane;
      const bool ok = r < cnt_amb;
      const unsigned m = __ballot_sync(0xffffffffu, ok);
      int b = 0;
      if (lane == 0) b = atomicAdd(ovf_count, __popc(m));
      b = __shfl_sync(0xffffffffu, b, 0);
      if (ok) ovf_list[b + __popc(m & ((1u << lane) - 1u))] = orig != nullptr ? orig[list[r]] : list[r];
    }
  }
  const int64_t cntA = bypassed ? 0 : cnt_amb;
  const int64_t cnt = cntA + cnt2;
  const int sub = lane & 7, grp = lane >> 3;
  const float brel = (float)(d + 8) * 0x1p-23f;
  const bool vec = (d & 3) == 0;
  const int d4 = d >> 2;
  for (int64_t rb = w0 * 4; rb < cnt; rb += nw * 4) {
    const int64_t r = rb + grp;
    const bool valid = r < cnt;
    const bool is2 = r >= cntA;
    const int64_t r2i = r - cntA;
    const int row = !valid ? 0 : is2 ? two_list[3 * r2i] : (orig != nullptr ? orig[list[r]] : list[r]);
    int nc = !valid ? 0 : is2 ? 2 : cand_n[r];
    const bool ovf = valid && (nc < 1 || nc > SB_NCAND);
    const unsigned om = __ballot_sync(0xffffffffu, ovf && sub == 0);
    if (om) {
      int b = 0;
      if (lane == 0) b = atomicAdd(ovf_count, __popc(om));
      b = __shfl_sync(0xffffffffu, b, 0);
      if (ovf && sub == 0) ovf_list[b + __popc(om & ((1u << lane) - 1u))] = row;
    }
    if (ovf) nc = 0;
    const int ncmax = __reduce_max_sync(0xffffffffu, nc);
    auto cand_id = [&](int c) -> int { return is2 ? two_list[3 * r2i + 1 + c] : cand[r * SB_NCAND + c]; };
    const float* prow = P + (int64_t)row * d;
    float f1 = 3.4e38f, f2 = 3.4e38f;
    int bj = -1;
    for (int c = 0; c < ncmax; c += 2) {
      const int ja = c < nc ? cand_id(c) : -1, jb = c + 1 < nc ? cand_id(c + 1) : -1;
      const float* ra = C + (int64_t)(ja >= 0 ? ja : 0) * d;
      const float* rb2 = C + (int64_t)(jb >= 0 ? jb : (ja >= 0 ? ja : 0)) * d;
      float sa = 0.0f, sb = 0.0f;
      if (ja >= 0) {
        if (vec) {
          const float4* p4 = reinterpret_cast<const float4*>(prow);
          const float4* a4 = reinterpret_cast<const float4*>(ra);
          const float4* b4 = reinterpret_cast<const float4*>(rb2);
          for (int f0 = sub; f0 < d4; f0 += 32) {
            float4 x[4], ya[4], yb[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int f = f0 + 8 * u;
              const bool ok = f < d4;
              x[u] = ok ? __ldg(p4 + f) : make_float4(0, 0, 0, 0);
              ya[u] = ok ? __ldg(a4 + f) : make_float4(0, 0, 0, 0);
              yb[u] = ok ? __ldg(b4 + f) : make_float4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              sa = dist4f(x[u], ya[u], sa);
              sb = dist4f(x[u], yb[u], sb);
            }
          }
        } else {
          for (int t = sub; t < d; t += 8) {
            const float x = prow[t];
            const float ea = x - ra[t], eb = x - rb2[t];
            sa = fmaf(ea, ea, sa);
            sb = fmaf(eb, eb, sb);
          }
        }
      }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        sa += __shfl_xor_sync(0xffffffffu, sa, o);
        sb += __shfl_xor_sync(0xffffffffu, sb, o);
      }
      if (ja >= 0) {
        if (sa < f1) { f2 = f1; f1 = sa; bj = ja; } else if (sa < f2) { f2 = sa; }
      }
      if (jb >= 0) {
        if (sb < f1) { f2 = f1; f1 = sb; bj = jb; } else if (sb < f2) { f2 = sb; }
      }
    }
    const bool unsure = nc > 1 && f2 * (1.0f - brel) <= f1 * (1.0f + brel);
    if (__any_sync(0xffffffffu, unsure)) {
      double best = 0.0;
      int bj64 = -1;
      for (int c = 0; c < ncmax; ++c) {
        const int j = (unsure && c < nc) ? cand_id(c) : -1;
        double s64 = 0.0;
        if (j >= 0)
          for (int t = sub; t < d; t += 8) {
            const double e = (double)prow[t] - (double)C[(int64_t)j * d + t];
            s64 = fma(e, e, s64);
          }
        s64 += __shfl_xor_sync(0xffffffffu, s64, 4);
        s64 += __shfl_xor_sync(0xffffffffu, s64, 2);
        s64 += __shfl_xor_sync(0xffffffffu, s64, 1);
        if (j >= 0 && (bj64 < 0 || s64 < best || (s64 == best && j < bj64))) { best = s64; bj64 = j; }
      }
      if (unsure) bj = bj64;
    }
    if (sub == 0 && bj >= 0) labels[row] = bj;
  }
}

// Exact f64 distances of each ambiguous row to its candidates (8 lanes per
// row, 4 rows per warp), argmin with the lowest index on ties; rows without a
// usable candidate list (too many candidates, or the bypass) are appended to
// the overflow list for the 3xTF32 resolver.
template <int DQ>
#ifndef PCB_EX_MINB
#define PCB_EX_MINB 3  // measured at c3: 3 blocks (85 regs, no spills) beat 4 (64 regs, spills) and 2
#endif
__global__ void __launch_bounds__(256, DQ <= 4 ? PCB_EX_MINB : 2)  // latency-bound: many warps per SM
screen_exact_kernel(const float* __restrict__ P, int d, const float* __restrict__ C,
                    const int* __restrict__ list, const int* __restrict__ count, int64_t bypass,
                    const int* __restrict__ cand, const int* __restrict__ cand_n, int32_t* __restrict__ labels,
                    int* __restrict__ ovf_list, int* __restrict__ ovf_count, const int32_t* __restrict__ orig,
                    const int* __restrict__ two_list, const int* __restrict__ two_count,
                    const long long* __restrict__ state) {
  if (stopped(state)) return;
  const int64_t cnt_amb = *count;
  const int64_t cnt2 = two_count != nullptr ? *two_count : 0;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool bypassed = cnt_amb > bypass;
  if (bypassed) {
    // bypass: the whole pass-1 list goes to the 3xTF32 resolver (32 entries per warp)
    for (int64_t b0 = w0 * 32; b0 < cnt_amb; b0 += nw * 32) {
      const int64_t r = b0 + lane;
      const bool ok = r < cnt_amb;
      const unsigned m = __ballot_sync(0xffffffffu, ok);
      int b = 0;
      if (lane == 0) b = atomicAdd(ovf_count, __popc(m));
      b = __shfl_sync(0xffffffffu, b, 0);
      if (ok) ovf_list[b + __popc(m & ((1u << lane) - 1u))] = orig != nullptr ? orig[list[r]] : list[r];
    }
  }
  // rows [0, cntA): pass-2 candidate lists; [cntA, cntA + cnt2): two-candidate rows of pass 1
  const int64_t cntA = bypassed ? 0 : cnt_amb;
  const int64_t cnt = cntA + cnt2;
  const int sub = lane & 7, grp = lane >> 3;
  for (int64_t rb = w0 * 4; rb < cnt; rb += nw * 4) {
    const int64_t r = rb + grp;
    const bool valid = r < cnt;
    const bool is2 = r >= cntA;
    const int64_t r2i = r - cntA;
    const int row = !valid ? 0 : is2 ? two_list[3 * r2i] : (orig != nullptr ? orig[list[r]] : list[r]);  // original id
    int nc = !valid ? 0 : is2 ? 2 : cand_n[r];
    const bool ovf = valid && (nc < 1 || nc > SB_NCAND);
    const unsigned om = __ballot_sync(0xffffffffu, ovf && sub == 0);
    if (om) {  // one atomic per warp
      int b = 0;
      if (lane == 0) b = atomicAdd(ovf_count, __popc(om));
      b = __shfl_sync(0xffffffffu, b, 0);
      if (ovf && sub == 0) ovf_list[b + __popc(om & ((1u << lane) - 1u))] = row;
    }
    if (ovf) nc = 0;
    const int ncmax = __reduce_max_sync(0xffffffffu, nc);
    // all candidate ids at once (two 16-byte loads), the point row as float4
    // candidate ids straight from the lists (L2) as the loop needs them
    auto cand_id = [&](int c) -> int {
      return is2 ? two_list[3 * r2i + 1 + c] : cand[r * SB_NCAND + c];
    };
    float4 p[DQ];
#pragma unroll
    for (int q = 0; q < DQ; ++q) p[q] = nc > 0 ? load4(P + (int64_t)row * d, sub + 8 * q, d) : make_float4(0, 0, 0, 0);
    // f32 distances first: sum (p - c)^2 has relative error <= (d + 8) 2^-23
    // (positive terms); the winner is certain unless the runner-up is within
    // that margin — then (rarely) the row is redone in f64, ties included
    const float brel = (float)(d + 8) * 0x1p-23f;
    float f1 = 3.4e38f, f2 = 3.4e38f;
    int bj = -1;
    for (int c = 0; c < ncmax; c += 2) {
      const int ja = c < nc ? cand_id(c) : -1, jb = c + 1 < nc ? cand_id(c + 1) : -1;
      float4 xa[DQ], xb[DQ];
#pragma unroll
      for (int q = 0; q < DQ; ++q) {
        xa[q] = ja >= 0 ? load4(C + (int64_t)ja * d, sub + 8 * q, d) : make_float4(0, 0, 0, 0);
        xb[q] = jb >= 0 ? load4(C + (int64_t)jb * d, sub + 8 * q, d) : make_float4(0, 0, 0, 0);
      }
      float sa = 0.0f, sb = 0.0f;
#pragma unroll
      for (int q = 0; q < DQ; ++q) {
        sa = dist4f(p[q], xa[q], sa);
        sb = dist4f(p[q], xb[q], sb);
      }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        sa += __shfl_xor_sync(0xffffffffu, sa, o);
        sb += __shfl_xor_sync(0xffffffffu, sb, o);
      }
      if (ja >= 0) {
        if (sa < f1) { f2 = f1; f1 = sa; bj = ja; } else if (sa < f2) { f2 = sa; }
      }
      if (jb >= 0) {
        if (sb < f1) { f2 = f1; f1 = sb; bj = jb; } else if (sb < f2) { f2 = sb; }
      }
    }
    const bool unsure = nc > 1 && f2 * (1.0f - brel) <= f1 * (1.0f + brel);
    if (__any_sync(0xffffffffu, unsure)) {
      // exact f64 pass for the rows whose f32 margin is too thin
      double best = 0.0;
      int bj64 = -1;
      for (int c = 0; c < ncmax; ++c) {
        const int j = (unsure && c < nc) ? cand_id(c) : -1;
        double s64 = 0.0;
        if (j >= 0) {
#pragma unroll
          for (int q = 0; q < DQ; ++q) s64 = dist4(p[q], load4(C + (int64_t)j * d, sub + 8 * q, d), s64);
        }
        s64 += __shfl_xor_sync(0xffffffffu, s64, 4);
        s64 += __shfl_xor_sync(0xffffffffu, s64, 2);
        s64 += __shfl_xor_sync(0xffffffffu, s64, 1);
        if (j >= 0 && (bj64 < 0 || s64 < best || (s64 == best && j < bj64))) { best = s64; bj64 = j; }
      }
      if (unsure) bj = bj64;
    }
    if (sub == 0 && bj >= 0) labels[row] = bj;
  }
}

}  // namespace pcb

using namespace pcb;

// Augmented B columns of centroid j: |c_j|^2 + OFF split into three BF16
// pieces (24 significant bits; the f32 key arithmetic allowance of the bound
// covers the rest), zeros after; padding rows j >= k get a huge key.
__global__ void centroid_aug_kernel(const float* __restrict__ cnorm, const float* __restrict__ bstat, int k, int kpad,
                                    __nv_bfloat16* __restrict__ aug) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= kpad) return;
  uint4 lo = make_uint4(0u, 0u, 0u, 0u), hi = make_uint4(0u, 0u, 0u, 0u);
  __nv_bfloat16 h1, h2, h3;
  if (j < k) {
    const float cp = (cnorm[j] + bstat[2]) * bstat[4];  // keys carry the operand scales S (E4M3; 1 for BF16)
    h1 = __float2bfloat16_rn(cp);
    const float r1 = cp - __bfloat162float(h1);  // exact (Sterbenz-like: |r1| << cp)
    h2 = __float2bfloat16_rn(r1);
    h3 = __float2bfloat16_rn(r1 - __bfloat162float(h2));
  } else {
    h1 = __float2bfloat16_rn(3.0e38f);
    h2 = h3 = __float2bfloat16_rn(0.0f);
  }
  lo.x = (uint32_t)__bfloat16_as_ushort(h1) | ((uint32_t)__bfloat16_as_ushort(h2) << 16);
  lo.y = (uint32_t)__bfloat16_as_ushort(h3);
  uint4* dst = reinterpret_cast<uint4*>(aug + (int64_t)j * SB_AUG);
  dst[0] = lo;
  dst[1] = hi;
}

extern "C" int pcb_screen_bf16_ld(int d) { return (d + SB_BKE - 1) / SB_BKE * SB_BKE; }
extern "C" int pcb_screen_bf16_ncand(void) { return SB_NCAND; }

extern "C" int pcb_screen_prep_points_bf16(const float* P, int64_t n, int d, int ldb, void* P_b, float* anorm,
                                           float* danorm, float* bstat, void* stream) {
  if (n < 1 || d < 1 || ldb < d || ldb % SB_BKE || !P || !P_b || !anorm || !danorm || !bstat) return PCB_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(bstat, 0, 4 * sizeof(float), st);
  if (e != cudaSuccess) return (int)e;
  const int grid = (int)std::min<int64_t>((n * 32 + 255) / 256, (int64_t)sm_count() * 16);
  row_bf16_norms_kernel<<<grid, 256, 0, st>>>(P, n, d, anorm, danorm, bstat + 3,
                                              reinterpret_cast<__nv_bfloat16*>(P_b), ldb);
  PCB_CHECK_LAUNCH();
  screen_off_kernel<<<1, 1, 0, st>>>(bstat, bstat + 3);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_screen_bf16_kpad(int k) { return (k + SB_KPAD - 1) / SB_KPAD * SB_KPAD; }
extern "C" int pcb_screen_bf16_aug(void) { return SB_AUG; }

extern "C" int pcb_screen_prep_centroids_bf16(const float* C, const float* cnorm, int k, int d, int ldb, void* C_b,
                                              void* C_aug, float* bnorm,
                                              float* dbnorm, float* bstat, void* stream) {
  if (k < 1 || d < 1 || ldb < d || ldb % SB_BKE || !C || !cnorm || !C_b || !C_aug || !bnorm || !dbnorm || !bstat)
    return PCB_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(bstat, 0, 2 * sizeof(float), st);
  if (e != cudaSuccess) return (int)e;
  // B operand rows are -2 bf16(c) (exact scaling): the MMA accumulates the key
  // |c|^2 + OFF - 2 <p~, c~> directly (centroid_aug_kernel supplies |c|^2 + OFF)
  row_bf16_norms_kernel<<<(k * 32 + 255) / 256, 256, 0, st>>>(C, k, d, bnorm, dbnorm, nullptr,
                                                             reinterpret_cast<__nv_bfloat16*>(C_b), ldb, -2.0f);
  PCB_CHECK_LAUNCH();
  const int kpad = (k + SB_KPAD - 1) / SB_KPAD * SB_KPAD;
  centroid_aug_kernel<<<(kpad + 127) / 128, 128, 0, st>>>(cnorm, bstat, k, kpad, reinterpret_cast<__nv_bfloat16*>(C_aug));
  PCB_CHECK_LAUNCH();
  max2_bf16_kernel<<<1, 256, 0, st>>>(bnorm, dbnorm, k, bstat);
  PCB_CHECK_LAUNCH();
  return 0;
}

// Pass 1 over all n rows: certified labels, ambiguous rows + thresholds.
extern "C" int pcb_assign_screen_bf16(const void* P_b, int64_t n, int ldb, const void* C_b, int k,
                                      const void* C_aug, const float* anorm, const float* danorm,
                                      const float* bstat, int32_t* labels, int* amb_list, int* amb_count,
                                      float* amb_thr, const int32_t* orig, const int32_t* labels_prev,
                                      int* two_list, int* two_count, const long long* state, void* stream) {
  if (n < 1 || ldb < SB_BKE || ldb % SB_BKE || k < 1 || !P_b || !C_b || !C_aug || !anorm || !danorm || !bstat ||
      !labels || !amb_list || !amb_count || !amb_thr)
    return PCB_EINVAL;
  if (n > INT32_MAX || k > SC_KMAX) return PCB_EUNSUP;
  return dispatch_bf16<false>(ldb, (const __nv_bfloat16*)P_b, n, (const __nv_bfloat16*)C_b, k, anorm, danorm,
                              (const __nv_bfloat16*)C_aug,
                              bstat, labels, amb_list, amb_count, amb_thr, 0, nullptr, nullptr, orig, labels_prev,
                              two_list, two_count, state,
                              (cudaStream_t)stream);
}

// Pass 2 + exact resolution of the ambiguous rows.  Rows left over (more than
// SB_NCAND candidates, or every row when the ambiguous count exceeds `bypass`)
// land in ovf_list / ovf_count for the 3xTF32 resolver.
// ldb in BF16 units (E4M3 rows: bytes / 2)
template <bool F8>
static int resolve_screen(const float* P, int64_t n, int d, const void* P_b, int ldb, const void* C_b,
                          const float* C, int k, const void* C_aug, const float* bstat,
                          const int* amb_list, const int* amb_count, const float* amb_thr,
                          int64_t bypass, void* sub_b, int* cand, int* cand_n, int32_t* labels,
                          int* ovf_list, int* ovf_count, const int32_t* orig, const int* two_list,
                          const int* two_count, const long long* state, void* stream) {
  if (n < 1 || d < 1 || k < 1 || (ldb % SB_BKE && !(F8 && ldb == 32)) || !P || !P_b || !C_b || !C || !C_aug || !bstat ||
      !amb_list || !amb_count || !amb_thr || !sub_b || !cand || !cand_n || !labels || !ovf_list || !ovf_count)
    return PCB_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(ovf_count, 0, sizeof(int), st);
  if (e != cudaSuccess) return (int)e;
  const int grid = sm_count() * 8;
  gather_rows_bf16<<<grid, 256, 0, st>>>((const __nv_bfloat16*)P_b, ldb, amb_list, amb_count, bypass,
                                         (__nv_bfloat16*)sub_b, state);
  PCB_CHECK_LAUNCH();
  int rc = dispatch_bf16<true, F8>(ldb, (const __nv_bfloat16*)sub_b, n, (const __nv_bfloat16*)C_b, k, nullptr, nullptr,
                               (const __nv_bfloat16*)C_aug, bstat, nullptr, nullptr, const_cast<int*>(amb_count),
                               const_cast<float*>(amb_thr), bypass, cand, cand_n, nullptr, nullptr, nullptr, nullptr,
                               state, st);
  if (rc) return rc;
  const int DQ = (d + 31) / 32;  // float4 per lane (8 lanes per row)
  const int xgrid = sm_count() * 4;  // ~one resident wave (grid-stride over the rows)
#define PCB_EX_CASE(N)                                                                                          \
  if (DQ <= N) {                                                                                              \
    screen_exact_kernel<N><<<xgrid, 256, 0, st>>>(P, d, C, amb_list, amb_count, bypass, cand, cand_n, labels, \
                                                  ovf_list, ovf_count, orig, two_list, two_count, state);     \
  } else
  PCB_EX_CASE(1)
  PCB_EX_CASE(2)
  PCB_EX_CASE(4)
  PCB_EX_CASE(8)
  screen_exact_wide_kernel<<<xgrid, 256, 0, st>>>(P, d, C, amb_list, amb_count, bypass, cand, cand_n, labels, ovf_list,
                                                  ovf_count, orig, two_list, two_count, state);
#undef PCB_EX_CASE
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_resolve_screen_bf16(const float* P, int64_t n, int d, const void* P_b, int ldb, const void* C_b,
                                       const float* C, int k, const void* C_aug, const float* bstat,
                                       const int* amb_list, const int* amb_count, const float* amb_thr,
                                       int64_t bypass, void* sub_b, int* cand, int* cand_n, int32_t* labels,
                                       int* ovf_list, int* ovf_count, const int32_t* orig, const int* two_list,
                                       const int* two_count, const long long* state, void* stream) {
  if (ldb < d) return PCB_EINVAL;
  return resolve_screen<false>(P, n, d, P_b, ldb, C_b, C, k, C_aug, bstat, amb_list, amb_count, amb_thr, bypass,
                               sub_b, cand, cand_n, labels, ovf_list, ovf_count, orig, two_list, two_count, state,
                               stream);
}

// Row layout of the screen's inputs: P_b[s] = Pb0[perm[s]] (256-byte BF16
// rows), anorm/danorm likewise, orig[s] = perm[s]; Pb0 / an0 / dan0 are the
// original-order copies written once by pcb_screen_prep_points_bf16 and perm
// is the point-id order of the last counting sort (pcb_sort_by_label).  Rows of
// one cluster become contiguous, so the rows of a screening warp share their
// nearest centroids and the epilogue's chunk skip fires; labels and the
// ambiguous-row resolution keep using original row ids.
__global__ void __launch_bounds__(256)
relayout_rows_bf16(const uint4* __restrict__ src, int per, const float* __restrict__ an0,
                   const float* __restrict__ dan0, const int32_t* __restrict__ perm, int64_t n, uint4* __restrict__ dst,
                   float* __restrict__ an, float* __restrict__ dan, int32_t* __restrict__ orig) {
  const int64_t total = n * per;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = e / per, q = e - s * per;
    const int64_t i = perm[s];
    dst[e] = __ldcs(src + i * per + q);
    if (q == 0) {
      an[s] = an0[i];
      dan[s] = dan0[i];
      orig[s] = (int32_t)i;
    }
  }
}

extern "C" int pcb_screen_relayout_bf16(const void* Pb0, const float* an0, const float* dan0, int64_t n, int ldb,
                                        const int32_t* perm, void* P_b, float* anorm, float* danorm, int32_t* orig,
                                        void* stream) {
  if (n < 1 || ldb < 8 || ldb % 8 || !Pb0 || !an0 || !dan0 || !perm || !P_b || !anorm || !danorm || !orig ||
      Pb0 == P_b)
    return PCB_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const int per = ldb / 8;  // 16-byte vectors per row
  const int grid = (int)std::min<int64_t>((n * per + 255) / 256, (int64_t)sm_count() * 32);
  relayout_rows_bf16<<<grid, 256, 0, st>>>(reinterpret_cast<const uint4*>(Pb0), per, an0, dan0, perm, n,
                                           reinterpret_cast<uint4*>(P_b), anorm, danorm, orig);
  PCB_CHECK_LAUNCH();
  return 0;
}

// ---- E4M3 screening ("fp8s"): same kernels, operands in E4M3 ---------------------
// One E4M3 pass (kind::f8f6f4, twice the BF16 rate) over p~ = e4m3(p sp) / sp
// and c~ = e4m3(-2 c sc) / (-2 sc), power-of-two scales sp, sc chosen on the
// device from max |p| (once) and max |c| (per update) so the largest entry maps
// to <= 448; the MMA emits keys scaled by S = sp sc (bstat[4]), the augmented
// BF16 step adds S (|c|^2 + OFF), and the bound (unscaled residual norms, E4M3
// half-ulp 2^-4) is scaled by S in the epilogue.  Rows are 128-byte chunks like
// the BF16 ones (viewed as BF16 pairs by the tensor maps).
__device__ __forceinline__ uint8_t to_e4m3(float x) {
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(x), "f"(x));
  return (uint8_t)(r & 0xFFu);
}
__device__ __forceinline__ float from_e4m3(uint8_t q) {
  uint32_t r;
  const uint16_t in = (uint16_t)q | (uint16_t)((uint16_t)q << 8);
  asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(r) : "h"(in));
  return __half2float(__ushort_as_half((unsigned short)(r & 0xFFFFu)));
}

__global__ void maxabs_kernel(const float* __restrict__ X, int64_t count, float* __restrict__ out) {
  float m = 0.0f;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, fabsf(X[e]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomic_max_pos_f(out, m);
}

// the largest power-of-two scale with m * scale <= 448 (E4M3 max finite)
__device__ __forceinline__ float e4m3_pow2_scale(float m) {
  float sc = 1.0f;
  if (m > 0.0f && isfinite(m)) {
    sc = exp2f(floorf(log2f(448.0f / m)));
    while (m * sc > 448.0f) sc *= 0.5f;
    while (m * sc * 2.0f <= 448.0f) sc *= 2.0f;
  }
  return sc;
}

// power-of-two scale with maxabs * mult * scale <= 448 (E4M3 max finite)
__global__ void e4m3_scale_kernel(const float* __restrict__ maxabs, float mult, float* __restrict__ scale,
                                  float* __restrict__ S, const float* __restrict__ other) {
  const float sc = e4m3_pow2_scale(*maxabs * mult);
  *scale = sc;
  if (S != nullptr) *S = sc * *other;
}

// The centroids' E4M3 scale, fixed for the fit: every coordinate of a mean of
// rows is within max |p| (bstat[6]), so sc = scale of 2 max |p| never
// saturates the rows e4m3(-2 c sc); centroids given by the caller that exceed
// it saturate (satfinite), which the exact residual norms |c - c~| charge to
// the bound.  S = sp sc.
__global__ void e4m3_centroid_scale_kernel(float* __restrict__ bstat) {
  const float sc = e4m3_pow2_scale(2.0f * bstat[6]);
  bstat[8] = sc;
  bstat[4] = sc * bstat[5];
}

// max |c~|, max |dc| over the centroids (bstat[0], bstat[1]) and the augmented
// columns S (|c|^2 + OFF) in three BF16 pieces (padding rows j >= k: huge key),
// one block: the tail of the per-iteration E4M3 centroid prep.
__global__ void __launch_bounds__(1024) centroid_max_aug_kernel(const float* __restrict__ bnorm,
                                                                const float* __restrict__ dbnorm,
                                                                const float* __restrict__ cnorm,
                                                                float* __restrict__ bstat, int k, int kpad,
                                                                __nv_bfloat16* __restrict__ aug) {
  __shared__ float red[32][2];
  float a = 0.0f, b = 0.0f;
  for (int j = threadIdx.x; j < k; j += blockDim.x) { a = fmaxf(a, bnorm[j]); b = fmaxf(b, dbnorm[j]); }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
    b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, o));
  }
  if ((threadIdx.x & 31) == 0) { red[threadIdx.x >> 5][0] = a; red[threadIdx.x >> 5][1] = b; }
  const float off = bstat[2], S = bstat[4];
  for (int j = threadIdx.x; j < kpad; j += blockDim.x) {
    uint4 lo = make_uint4(0u, 0u, 0u, 0u), hi = make_uint4(0u, 0u, 0u, 0u);
    __nv_bfloat16 h1, h2, h3;
    if (j < k) {
      const float cp = (cnorm[j] + off) * S;
      h1 = __float2bfloat16_rn(cp);
      const float r1 = cp - __bfloat162float(h1);  // exact
      h2 = __float2bfloat16_rn(r1);
      h3 = __float2bfloat16_rn(r1 - __bfloat162float(h2));
    } else {
      h1 = __float2bfloat16_rn(3.0e38f);
      h2 = h3 = __float2bfloat16_rn(0.0f);
    }
    lo.x = (uint32_t)__bfloat16_as_ushort(h1) | ((uint32_t)__bfloat16_as_ushort(h2) << 16);
    lo.y = (uint32_t)__bfloat16_as_ushort(h3);
    uint4* dst = reinterpret_cast<uint4*>(aug + (int64_t)j * SB_AUG);
    dst[0] = lo;
    dst[1] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { a = fmaxf(a, red[w][0]); b = fmaxf(b, red[w][1]); }
    a = fmaxf(a, red[0][0]);
    b = fmaxf(b, red[0][1]);
    bstat[0] = a;
    bstat[1] = b;
  }
}

// Per row: E4M3 copy of mult * scale * x (row stride ld8 bytes, zero padded),
// |x~| and |x - x~| (unscaled, rounded up), max |x|^2.
__global__ void __launch_bounds__(256)
row_e4m3_norms_kernel(const float* __restrict__ X, int64_t rows, int d, float* __restrict__ an, float* __restrict__ dan,
                      float* __restrict__ maxsq, uint8_t* __restrict__ Xq, int ld8, const float* __restrict__ scale,
                      float mult) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const float s = *scale * mult, inv = 1.0f / s;  // exact: powers of two
  float wmax = 0.0f;
  for (int64_t i = w; i < rows; i += nw) {
    double s_t = 0.0, s_d = 0.0, s_x = 0.0;
    for (int t = lane; t < ld8; t += 32) {
      const float x = t < d ? X[i * d + t] : 0.0f;
      const uint8_t q = to_e4m3(x * s);
      Xq[i * ld8 + t] = q;
      const double h = (double)(from_e4m3(q) * inv);
      const double dd = (double)x - h;
      s_t = fma(h, h, s_t);
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
  if (lane == 0 && maxsq != nullptr) atomic_max_pos_f(maxsq, wmax);
}

extern "C" int pcb_screen_fp8_ld(int d) { return d <= 64 ? 64 : (d + 127) / 128 * 128; }

// bstat (16 floats): [0] max|c~| [1] max|dc| [2] OFF [3] scratch [4] S = sp sc
// [5] sp [6] max|p| [7] (unused) [8] sc (the centroids' scale, fixed per fit from max|p|)
extern "C" int pcb_screen_prep_points_fp8(const float* P, int64_t n, int d, int ld8, void* P_q, float* anorm,
                                          float* danorm, float* bstat, void* stream) {
  if (n < 1 || d < 1 || ld8 < d || (ld8 % 128 && ld8 != 64) || !P || !P_q || !anorm || !danorm || !bstat)
    return PCB_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(bstat, 0, 16 * sizeof(float), st);
  if (e != cudaSuccess) return (int)e;
  const int g1 = (int)std::min<int64_t>((n * d + 255) / 256, (int64_t)sm_count() * 16);
  maxabs_kernel<<<g1, 256, 0, st>>>(P, n * d, bstat + 6);
  PCB_CHECK_LAUNCH();
  e4m3_scale_kernel<<<1, 1, 0, st>>>(bstat + 6, 1.0f, bstat + 5, nullptr, nullptr);
  PCB_CHECK_LAUNCH();
  const int grid = (int)std::min<int64_t>((n * 32 + 255) / 256, (int64_t)sm_count() * 16);
  row_e4m3_norms_kernel<<<grid, 256, 0, st>>>(P, n, d, anorm, danorm, bstat + 3, (uint8_t*)P_q, ld8, bstat + 5, 1.0f);
  PCB_CHECK_LAUNCH();
  screen_off_kernel<<<1, 1, 0, st>>>(bstat, bstat + 3);
  PCB_CHECK_LAUNCH();
  e4m3_centroid_scale_kernel<<<1, 1, 0, st>>>(bstat);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_screen_prep_centroids_fp8(const float* C, const float* cnorm, int k, int d, int ld8, void* C_q,
                                             void* C_aug, float* bnorm, float* dbnorm, float* bstat, void* stream) {
  if (k < 1 || d < 1 || ld8 < d || (ld8 % 128 && ld8 != 64) || !C || !cnorm || !C_q || !C_aug || !bnorm || !dbnorm ||
      !bstat)
    return PCB_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  // sc (bstat[8]) and S (bstat[4]) were fixed by pcb_screen_prep_points_fp8
  row_e4m3_norms_kernel<<<(k * 32 + 255) / 256, 256, 0, st>>>(C, k, d, bnorm, dbnorm, nullptr, (uint8_t*)C_q, ld8,
                                                             bstat + 8, -2.0f);
  PCB_CHECK_LAUNCH();
  const int kpad = (k + SB_KPAD - 1) / SB_KPAD * SB_KPAD;
  centroid_max_aug_kernel<<<1, 1024, 0, st>>>(bnorm, dbnorm, cnorm, bstat, k, kpad,
                                              reinterpret_cast<__nv_bfloat16*>(C_aug));
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_assign_screen_fp8(const void* P_q, int64_t n, int ld8, const void* C_q, int k, const void* C_aug,
                                     const float* anorm, const float* danorm, const float* bstat, int32_t* labels,
                                     int* amb_list, int* amb_count, float* amb_thr, const int32_t* orig,
                                     const int32_t* labels_prev, int* two_list, int* two_count,
                                     const long long* state, void* stream) {
  if (n < 1 || ld8 < 64 || (ld8 % 128 && ld8 != 64) || k < 1 || !P_q || !C_q || !C_aug || !anorm || !danorm ||
      !bstat || !labels ||
      !amb_list || !amb_count || !amb_thr)
    return PCB_EINVAL;
  if (n > INT32_MAX) return PCB_EUNSUP;
  return dispatch_bf16<false, true>(ld8 / 2, (const __nv_bfloat16*)P_q, n, (const __nv_bfloat16*)C_q, k, anorm,
                                    danorm, (const __nv_bfloat16*)C_aug, bstat, labels, amb_list, amb_count, amb_thr,
                                    0, nullptr, nullptr, orig, labels_prev, two_list, two_count, state,
                                    (cudaStream_t)stream);
}

extern "C" int pcb_resolve_screen_fp8(const float* P, int64_t n, int d, const void* P_q, int ld8, const void* C_q,
                                      const float* C, int k, const void* C_aug, const float* bstat,
                                      const int* amb_list, const int* amb_count, const float* amb_thr,
                                      int64_t bypass, void* sub_q, int* cand, int* cand_n, int32_t* labels,
                                      int* ovf_list, int* ovf_count, const int32_t* orig, const int* two_list,
                                      const int* two_count, const long long* state, void* stream) {
  if (ld8 < 64 || (ld8 % 128 && ld8 != 64) || ld8 < d) return PCB_EINVAL;
  return resolve_screen<true>(P, n, d, P_q, ld8 / 2, C_q, C, k, C_aug, bstat, amb_list, amb_count, amb_thr, bypass,
                              sub_q, cand, cand_n, labels, ovf_list, ovf_count, orig, two_list, two_count, state,
                              stream);
}
