// Probe: the screen kernel's accumulator handshake without data movement.
// One CTA per SM, 384 threads: warp 0 issues per centroid tile and row tile
// (2 row tiles) KS E4M3 K=32 MMAs + one BF16 K=16 augmented MMA into one of
// NB accumulators per row tile (N = 128 / NB... columns: 512 / (2 NB) each),
// commits to tfull; the 8 "epilogue" warps (4 per row tile) wait tfull,
// optionally load their 32 lanes x N columns (LD), and release tempty.
// Reported: SM0 clocks per tile (both row tiles), against the same MMAs
// issued back to back with no handshake.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a scripts/handshake_probe.cu -o /tmp/hs
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2501_05587_b200/csrc/tc_ptx.cuh"

using namespace pcb;

__device__ unsigned int* g_hang_host = nullptr;
__device__ __forceinline__ void wait_wd(uint64_t* bar, uint32_t parity, unsigned code) {
  const long long t0 = clock64();
  while (true) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(ptx::smem_u32(bar)), "r"(parity) : "memory");
    if (ok) return;
    if (clock64() - t0 > (1ll << 32)) {
      if (g_hang_host != nullptr) {
        atomicMax(g_hang_host, code);
        g_hang_host[1 + (code % 16)] = parity | (blockIdx.x << 8);
        __threadfence_system();
      }
      asm volatile("trap;");
    }
  }
}

__device__ __forceinline__ void umma_bf16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   ptx::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(ptx::smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld_x64(uint32_t taddr, uint32_t (&r)[64]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63]) : "r"(taddr));
}
__device__ __forceinline__ void tie64(uint32_t (&r)[64]) {
#pragma unroll
  for (int i = 0; i < 64; ++i) asm volatile("" : "+r"(r[i]));
}

// TMA: centroid tiles (KS * 32 B rows + the 4 KB augmented block) streamed from
// global memory (32 tiles, L2-resident) through a 4-stage ring by warp 3
// ARR: arrivals per release: 128 (every thread) or 4 (one lane per warp)
// HS: 0 = no handshake (MMAs back to back), 1 = handshake
// LD: 0 none; 1 chunk pairs, two waits, release after the second; 2 all four
// chunks, one wait, release, then use.  SPLIT: row tile r's MMAs issued by warp r
// (TMA 6 only; the ring stage released by one epilogue lane per row tile)
template <int KS, int NB, int N, int ARR, int LD, bool HS, int TMA = 0, bool SPLIT = false>
__global__ void __launch_bounds__(384, 1) probe(int tiles, unsigned long long* cycles, const uint8_t* Bg) {
  constexpr int STAGES = 4;
  constexpr uint32_t kB = 128 * KS * 32, kStage = kB + 4096;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw & 1023u)) & 1023u);
  uint8_t* sA = smem;            // 2 row tiles x 16 KB
  uint8_t* sB = smem + 32768;    // 4 stages x 16 KB
  uint8_t* sX = smem + 98304;    // augmented operands
  __shared__ uint64_t tfull[2 * NB], tempty[2 * NB], done, full[STAGES], empty[STAGES], dummy, done2;
  uint8_t* sR = smem + 106496;   // TMA ring
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 106496 / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u;
    h ^= h >> 15;
    h *= 0x85ebca6bu;
    h ^= h >> 13;
    reinterpret_cast<uint32_t*>(smem)[i] = h & 0x37373737u;
  }
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2 * NB; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], ARR);
    }
    ptx::mbar_init(&done, SPLIT ? 2 : 1);
    ptx::mbar_init(&dummy, 1);
    ptx::mbar_init(&done2, 1);
    ptx::mbar_arrive(&done2);  // phase 0 complete
    for (int i = 0; i < STAGES; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], SPLIT ? 2 : 1);
    }
    ptx::fence_barrier_init();
  }
  if (threadIdx.x < 32) ptx::tmem_alloc<512>(&tslot);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 || (SPLIT && warp == 1)) {
    const uint32_t idesc_8 = ptx::idesc_e4m3<128, N>();
    const uint32_t idesc_h = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t bb = ptx::sdesc_k_sw128(ptx::smem_u32(sB));
    const uint64_t aa = ptx::sdesc_k_none(ptx::smem_u32(sX), 128 * 16, 128);
    const uint64_t ba = ptx::sdesc_k_none(ptx::smem_u32(sX + 4096), N * 16, 128);
    const unsigned long long t0 = clock64();
    int buf = 0;
    uint32_t ph = 0;
    int stage = 0;
    uint32_t sph = 0;
    for (int t = 0; t < tiles; ++t) {
      uint64_t bs = bb + (uint64_t)(((t & 3) * 16384) >> 4);
      if (TMA == 5) ptx::mbar_wait(&done2, 0);
      if ((TMA >= 1 && TMA <= 3) || TMA == 6) {
        ptx::mbar_wait(&full[stage], sph);
        if (TMA != 2) bs = (KS == 4 ? ptx::sdesc_k_sw128(ptx::smem_u32(sR + stage * kStage))
                      : ptx::sdesc_k_sw64(ptx::smem_u32(sR + stage * kStage)));
      }
      for (int rt = SPLIT ? warp : 0; rt < (SPLIT ? warp + 1 : 2); ++rt) {
        if (HS) ptx::mbar_wait(&tempty[buf * 2 + rt], ph ^ 1u);
        ptx::tc_fence_after();
        const uint32_t d = tmem + (uint32_t)((buf * 2 + rt) * N);
        const uint64_t a = ptx::sdesc_k_sw128(ptx::smem_u32(sA + rt * 16384));
        if (ptx::elect_one()) {
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) {
            const uint64_t off = (uint64_t)(ks * 32) >> 4;
            ptx::umma_f8(d, a + off, bs + off, idesc_8, ks != 0);
          }
          umma_bf16(d, aa, ba, idesc_h, 1u);
          if (HS) ptx::umma_commit(&tfull[buf * 2 + rt]);
          if (TMA >= 1 && TMA <= 3 && rt == 1) ptx::umma_commit(&empty[stage]);
          if (TMA == 4 && rt == 1) ptx::umma_commit(&dummy);
        }
        __syncwarp();
      }
      if (++buf == NB) { buf = 0; ph ^= 1u; }
      if (++stage == STAGES) { stage = 0; sph ^= 1u; }
    }
    if (ptx::elect_one()) ptx::umma_commit(&done);
    __syncwarp();
    ptx::mbar_wait(&done, 0);
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    if (SPLIT && threadIdx.x == 32) cycles[blockIdx.x] = max(cycles[blockIdx.x], t1 - t0);
  } else if (warp == 3 && ((TMA >= 1 && TMA <= 3) || TMA == 6)) {
    int stage = 0;
    uint32_t sph = 0;
    for (int t = 0; t < tiles; ++t) {
      ptx::mbar_wait(&empty[stage], sph ^ 1u);
      if (ptx::elect_one()) {
        const int tile = t & 31;
        uint8_t* st = sR + stage * kStage;
        if (TMA == 3 || TMA == 6) {
          ptx::mbar_arrive(&full[stage]);
        } else {
        ptx::mbar_expect_tx(&full[stage], kStage);
        bulk_g2s(st, Bg + (size_t)tile * kB, kB, &full[stage]);
        bulk_g2s(st + kB, Bg + 32 * (size_t)kB + tile * 4096, 2048, &full[stage]);
        bulk_g2s(st + kB + 2048, Bg + 32 * (size_t)kB + tile * 4096 + 2048, 2048, &full[stage]);
        }
      }
      __syncwarp();
      if (++stage == STAGES) { stage = 0; sph ^= 1u; }
    }
  } else if (warp >= 4 && HS) {
    const int g = warp & 3, h = (warp - 4) >> 2;
    int buf = 0;
    uint32_t ph = 0;
    for (int t = 0; t < tiles; ++t) {
      ptx::mbar_wait(&tfull[buf * 2 + h], ph);
      ptx::tc_fence_after();
      if (TMA == 6 && (SPLIT || h == 1) && g == 0 && lane == 0) ptx::mbar_arrive(&empty[t % STAGES]);
      if (LD == 3) {
        const uint32_t ta = tmem + ((uint32_t)(g * 32) << 16) + (uint32_t)((buf * 2 + h) * N);
        uint32_t r0[64], r1[64];
        tmem_ld_x64(ta, r0);
        tmem_ld_x64(ta + 64, r1);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        tie64(r0);
        tie64(r1);
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[buf * 2 + h]);
        uint32_t x = 0;
#pragma unroll
        for (int i = 0; i < 64; ++i) x ^= r0[i] ^ r1[i];
        if (x == 0x12345678u) asm volatile("trap;");
        if (++buf == NB) { buf = 0; ph ^= 1u; }
        continue;
      }
      if (LD == 2) {
        const uint32_t ta = tmem + ((uint32_t)(g * 32) << 16) + (uint32_t)((buf * 2 + h) * N);
        uint32_t r0[32], r1[32], r2[32], r3[32];
        ptx::tmem_ld_32x32b_x32_async(ta, r0);
        ptx::tmem_ld_32x32b_x32_async(ta + 32, r1);
        ptx::tmem_ld_32x32b_x32_async(ta + 64, r2);
        ptx::tmem_ld_32x32b_x32_async(ta + 96, r3);
        ptx::tmem_wait_ld(r0);
        ptx::tie_regs(r1);
        ptx::tie_regs(r2);
        ptx::tie_regs(r3);
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[buf * 2 + h]);
        uint32_t x = 0;
#pragma unroll
        for (int i = 0; i < 32; ++i) x ^= r0[i] ^ r1[i] ^ r2[i] ^ r3[i];
        if (x == 0x12345678u) asm volatile("trap;");
        if (++buf == NB) { buf = 0; ph ^= 1u; }
        continue;
      }
      if (LD) {
        const uint32_t ta = tmem + ((uint32_t)(g * 32) << 16) + (uint32_t)((buf * 2 + h) * N);
        uint32_t r0[32], r1[32];
#pragma unroll
        for (int q = 0; q < N / 32; q += 2) {
          ptx::tmem_ld_32x32b_x32_async(ta + 32 * q, r0);
          ptx::tmem_ld_32x32b_x32_async(ta + 32 * q + 32, r1);
          ptx::tmem_wait_ld(r0);
          ptx::tie_regs(r1);
          uint32_t x = 0;
#pragma unroll
          for (int i = 0; i < 32; ++i) x ^= r0[i] ^ r1[i];
          if (x == 0x12345678u) asm volatile("trap;");
        }
      }
      ptx::tc_fence_before();
      if (ARR == 128) ptx::mbar_arrive(&tempty[buf * 2 + h]);
      else {
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&tempty[buf * 2 + h]);
      }
      if (++buf == NB) { buf = 0; ph ^= 1u; }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 0) ptx::tmem_dealloc<512>(tmem);
}

template <int KS, int NB, int N, int ARR, int LD, bool HS, int TMA = 0, bool SPLIT = false>
static void run(int sms, int tiles, const char* name) {
  static uint8_t* Bg = nullptr;
  if (Bg == nullptr) {
    cudaMalloc(&Bg, 32 * (128 * 128 + 4096));
    cudaMemset(Bg, 0x11, 32 * (128 * 128 + 4096));
  }
  static_assert(2 * NB * N <= 512, "TMEM columns");
  unsigned long long* cyc;
  cudaMalloc(&cyc, sms * sizeof(unsigned long long));
  const int smem = 106496 + 4 * (128 * 128 + 4096) + 1024;
  auto k = probe<KS, NB, N, ARR, LD, HS, TMA, SPLIT>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<<<sms, 384, smem>>>(tiles / 10, cyc, Bg);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<sms, 384, smem>>>(tiles, cyc, Bg);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long c0;
  cudaMemcpy(&c0, cyc, sizeof(c0), cudaMemcpyDeviceToHost);
  // per 128 centroid columns (N = 64 tiles: two of them)
  printf("KS=%d NB=%d N=%3d arr=%3d ld=%d hs=%d tma=%d split=%d %-34s %8.1f clk per 128 cols x 2 row tiles (%.2f GHz eff)  %s\n", KS, NB,
         N, ARR, (int)LD, (int)HS, (int)TMA, (int)SPLIT, name, (double)c0 / tiles * (128 / N), (double)c0 / (ms * 1e6),
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  setvbuf(stdout, nullptr, _IONBF, 0);
  unsigned* hh;
  cudaHostAlloc(&hh, 17 * 4, cudaHostAllocMapped);
  for (int i = 0; i < 17; ++i) hh[i] = 0;
  unsigned* dh;
  cudaHostGetDevicePointer(&dh, hh, 0);
  cudaMemcpyToSymbol(g_hang_host, &dh, sizeof(dh));
  for (int r = 0; r < 2; ++r) {
    run<2, 2, 128, 128, 2, true, 6, true>(sms, 40000, "c5 split, ld x32 x4");
    run<2, 2, 128, 128, 3, true, 6, true>(sms, 40000, "c5 split, ld x64 x2");
    run<4, 2, 128, 128, 2, true, 6, true>(sms, 40000, "c3 split, ld x32 x4");
    run<4, 2, 128, 128, 3, true, 6, true>(sms, 40000, "c3 split, ld x64 x2");
  }
  for (int i = 0; i < 17; ++i) printf("%u ", hh[i]);
  printf(" <- hang codes\n");
  return 0;
}
