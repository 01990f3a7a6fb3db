// On-device init_assignments (clustering.py:91-108): the reference's labels,
// bit for bit, generated in HBM instead of on the host.
//
// The reference draws `Generator(PCG64(seed)).integers(0, k, size=n)` and then
// repeats {labels[j] = j for every empty cluster j} until no cluster is empty.
// numpy's algorithm for that draw (numpy 1.17+ and 2.x, int64 output, range
// k - 1 <= 0xFFFFFFFF, unmasked):
//   * seeding: SeedSequence(seed).generate_state(4, uint64) = [s0, s1, s2, s3];
//     pcg64_set_seed(initstate = s0:s1, initseq = s2:s3) (hi:lo 128-bit), i.e.
//     state = 0, inc = initseq << 1 | 1, step, state += initstate, step;
//   * PCG64 (XSL-RR 128/64): step state = state * M + inc, output
//     rotr64(hi ^ lo, hi >> 58) of the new state;
//   * next_uint32 splits each 64-bit output: low half first, then high half;
//   * Lemire's bounded draw: m = u32 * k, accept unless low32(m) < (2^32 - k) % k,
//     value = m >> 32; a rejected draw is replaced by the next u32.
// So label i is the i-th ACCEPTED 32-bit draw.  Rejections have probability
// < k / 2^32 (zero for powers of two), so the kernel writes draw i to label i
// and records rejected draw positions; a compaction pass (only when some draw
// was rejected) shifts the labels over them using the sorted rejection list.
// Each thread jumps ahead to its own block of the PCG64 stream (O(log n)
// 128-bit LCG advance), so generation is embarrassingly parallel.
#include "pcb_common.cuh"
#include "pcb_launch.cuh"

namespace pcb {

typedef unsigned __int128 u128;

__host__ __device__ __forceinline__ u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
}

__host__ __device__ __forceinline__ uint64_t pcg_output(u128 s) {
  const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  const uint64_t x = hi ^ lo;
  const unsigned rot = (unsigned)(hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

// state after `delta` LCG steps (Brown's jump-ahead)
__host__ __device__ inline u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = inc;
  while (delta > 0) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

// ---- numpy SeedSequence (bit_generator.pyx), host side ----------------------
namespace seedseq {
constexpr uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u, INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
constexpr uint32_t MIX_MULT_L = 0xca01f9ddu, MIX_MULT_R = 0x4973f715u;
constexpr int XSHIFT = 16, POOL = 4;
static inline uint32_t hashmix(uint32_t value, uint32_t& hc) {
  value ^= hc;
  hc *= MULT_A;
  value *= hc;
  value ^= value >> XSHIFT;
  return value;
}
static inline uint32_t mix(uint32_t x, uint32_t y) {
  uint32_t r = MIX_MULT_L * x - MIX_MULT_R * y;
  r ^= r >> XSHIFT;
  return r;
}
}  // namespace seedseq

// PCG64(seed) initial (state, inc) for a non-negative integer seed < 2^64.
static void pcg64_from_seed(uint64_t seed, u128* state, u128* inc) {
  using namespace seedseq;
  uint32_t ent[2];
  int nent = 0;
  // _coerce_to_uint32_array: little-endian 32-bit words, at least one word
  ent[nent++] = (uint32_t)seed;
  if (seed >> 32) ent[nent++] = (uint32_t)(seed >> 32);
  uint32_t pool[POOL];
  uint32_t hc = INIT_A;
  for (int i = 0; i < POOL; ++i) pool[i] = hashmix(i < nent ? ent[i] : 0u, hc);
  for (int s = 0; s < POOL; ++s)
    for (int d = 0; d < POOL; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s], hc));
  for (int s = POOL; s < nent; ++s)
    for (int d = 0; d < POOL; ++d) pool[d] = mix(pool[d], hashmix(ent[s], hc));
  // generate_state(4, uint64): 8 uint32 words, viewed as 4 little-endian u64
  uint32_t w[8];
  uint32_t hb = INIT_B;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i % POOL];
    v ^= hb;
    hb *= MULT_B;
    v *= hb;
    v ^= v >> XSHIFT;
    w[i] = v;
  }
  uint64_t s64[4];
  for (int i = 0; i < 4; ++i) s64[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
  const u128 initstate = ((u128)s64[0] << 64) | s64[1];
  const u128 initseq = ((u128)s64[2] << 64) | s64[3];
  u128 st = 0;
  const u128 in = (initseq << 1) | 1u;
  st = st * pcg_mult() + in;
  st += initstate;
  st = st * pcg_mult() + in;
  *state = st;
  *inc = in;
}

constexpr int kOutPerThread = 32;  // 64-bit outputs per thread = 64 draws

// Draw j (0-based) of the 32-bit stream -> labels[j] (j < n) or extra[j - n].
__global__ void __launch_bounds__(256)
init_draw_kernel(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t n, int64_t ndraw,
                 uint32_t k, uint32_t threshold, int32_t* __restrict__ labels, int32_t* __restrict__ extra,
                 int64_t* __restrict__ rej, int* __restrict__ rej_count, int rej_cap) {
  const u128 state0 = ((u128)st_hi << 64) | st_lo, inc = ((u128)inc_hi << 64) | inc_lo;
  const int64_t nout = (ndraw + 1) / 2;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t o0 = t * kOutPerThread;
  if (o0 >= nout) return;
  u128 s = pcg_advance(state0, inc, (uint64_t)o0);
  const u128 M = pcg_mult();
  for (int q = 0; q < kOutPerThread; ++q) {
    const int64_t o = o0 + q;
    if (o >= nout) break;
    s = s * M + inc;
    const uint64_t x = pcg_output(s);
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int64_t j = 2 * o + half;
      if (j >= ndraw) break;
      const uint32_t u = half ? (uint32_t)(x >> 32) : (uint32_t)x;
      const uint64_t m = (uint64_t)u * k;
      const int32_t v = (int32_t)(m >> 32);
      if (j < n) labels[j] = v;
      else extra[j - n] = v;
      if ((uint32_t)m < threshold) {
        const int p = atomicAdd(rej_count, 1);
        if (p < rej_cap) rej[p] = j;
      }
    }
  }
}

// rank sort of the (few) rejected positions, one block; a[r] = q_r - r is the
// number of accepted draws before the r-th rejection
__global__ void __launch_bounds__(1024)
init_sort_rejections(const int64_t* __restrict__ rej, int R, int64_t* __restrict__ a) {
  for (int i = threadIdx.x; i < R; i += blockDim.x) {
    const int64_t v = rej[i];
    int r = 0;
    for (int j = 0; j < R; ++j) r += rej[j] < v;  // positions are distinct
    a[r] = v - r;
  }
}

// out[i] = draw (i + #{r : a[r] <= i})
__global__ void init_compact_kernel(const int32_t* __restrict__ labels, const int32_t* __restrict__ extra,
                                    int64_t n, const int64_t* __restrict__ a, int R, int32_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = R;  // first r with a[r] > i
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (a[mid] <= i) lo = mid + 1;
      else hi = mid;
    }
    const int64_t j = i + lo;
    out[i] = j < n ? labels[j] : extra[j - n];
  }
}

__global__ void init_hist_kernel(const int32_t* __restrict__ labels, int64_t n, int k, int* __restrict__ counts) {
  extern __shared__ int h[];
  for (int j = threadIdx.x; j < k; j += blockDim.x) h[j] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&h[labels[i]], 1);
  __syncthreads();
  for (int j = threadIdx.x; j < k; j += blockDim.x)
    if (h[j]) atomicAdd(&counts[j], h[j]);
}

__global__ void init_hist_global_kernel(const int32_t* __restrict__ labels, int64_t n, int* __restrict__ counts) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&counts[labels[i]], 1);
}

// labels[hollow] = hollow for every empty cluster (clustering.py:104-107)
__global__ void init_fill_hollow(const int* __restrict__ counts, int k, int32_t* __restrict__ labels,
                                 int* __restrict__ flag) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x)
    if (counts[j] == 0) {
      labels[j] = j;
      *flag = 1;
    }
}

struct InitScratch {
  int64_t extra_n, rej_cap;
  size_t off_extra, off_rej, off_a, off_tmp, off_counts, off_small, total;
};

static InitScratch init_layout(int64_t n, int k) {
  InitScratch s{};
  // expected rejections < n k / 2^32; the margin makes running short
  // (a PCB_EUNSUP return) astronomically unlikely
  const double expect = (double)n * (double)k / 4294967296.0;
  s.extra_n = 4096 + (int64_t)(16.0 * expect);
  s.rej_cap = s.extra_n;
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  size_t o = 0;
  s.off_extra = o; o = al(o + sizeof(int32_t) * s.extra_n);
  s.off_rej = o;   o = al(o + sizeof(int64_t) * s.rej_cap);
  s.off_a = o;     o = al(o + sizeof(int64_t) * s.rej_cap);
  s.off_tmp = o;   o = al(o + sizeof(int32_t) * (size_t)n);
  s.off_counts = o; o = al(o + sizeof(int) * (size_t)k);
  s.off_small = o; o = al(o + 4 * sizeof(int));
  s.total = o;
  return s;
}

}  // namespace pcb

using namespace pcb;

extern "C" int64_t pcb_init_scratch_bytes(int64_t n, int k) {
  if (n < 1 || k < 1) return PCB_EINVAL;
  return (int64_t)init_layout(n, k).total;
}

extern "C" int pcb_pcg64_seed_state(uint64_t seed, uint64_t* out4) {
  if (!out4) return PCB_EINVAL;
  u128 st, inc;
  pcg64_from_seed(seed, &st, &inc);
  out4[0] = (uint64_t)(st >> 64);
  out4[1] = (uint64_t)st;
  out4[2] = (uint64_t)(inc >> 64);
  out4[3] = (uint64_t)inc;
  return 0;
}

extern "C" int pcb_bounded_draws(int64_t n, int k, uint64_t seed, int32_t* out, void* scratch,
                                 int64_t scratch_bytes, void* stream) {
  if (n < 1 || k < 1 || !out || !scratch) return PCB_EINVAL;
  const InitScratch L = init_layout(n, k);
  if (scratch_bytes < (int64_t)L.total) return PCB_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* base = (uint8_t*)scratch;
  int32_t* extra = (int32_t*)(base + L.off_extra);
  int64_t* rej = (int64_t*)(base + L.off_rej);
  int64_t* a = (int64_t*)(base + L.off_a);
  int32_t* tmp = (int32_t*)(base + L.off_tmp);
  int* small = (int*)(base + L.off_small);  // [0] rejections
  u128 s0, inc;
  pcg64_from_seed(seed, &s0, &inc);
  const uint32_t kk = (uint32_t)k;
  const uint32_t threshold = (uint32_t)((0xFFFFFFFFu - (kk - 1u)) % kk);  // (UINT32_MAX - rng) % (rng + 1)
  const int64_t ndraw = n + L.extra_n;
  cudaError_t e = cudaMemsetAsync(small, 0, 4 * sizeof(int), st);
  if (e != cudaSuccess) return (int)e;
  const int64_t threads = ((ndraw + 1) / 2 + kOutPerThread - 1) / kOutPerThread;
  init_draw_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(
      (uint64_t)(s0 >> 64), (uint64_t)s0, (uint64_t)(inc >> 64), (uint64_t)inc, n, ndraw, kk, threshold, out,
      extra, rej, small, (int)L.rej_cap);
  PCB_CHECK_LAUNCH();
  int R = 0;
  if ((e = cudaMemcpyAsync(&R, small, sizeof(int), cudaMemcpyDeviceToHost, st)) != cudaSuccess) return (int)e;
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return (int)e;
  if (R > L.rej_cap || R > L.extra_n) return PCB_EUNSUP;
  if (R > 0) {
    init_sort_rejections<<<1, 1024, 0, st>>>(rej, R, a);
    PCB_CHECK_LAUNCH();
    const int grid = (int)std::min<int64_t>((n + 255) / 256, 4L * sm_count());
    init_compact_kernel<<<grid, 256, 0, st>>>(out, extra, n, a, R, tmp);
    PCB_CHECK_LAUNCH();
    if ((e = cudaMemcpyAsync(out, tmp, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
      return (int)e;
  }
  return 0;
}

extern "C" int pcb_init_assignments(int64_t n, int k, uint64_t seed, int32_t* labels, void* scratch,
                                    int64_t scratch_bytes, int* passes_out, void* stream) {
  if (n < 1 || k < 1 || k > n || !labels || !scratch) return PCB_EINVAL;
  const InitScratch L = init_layout(n, k);
  if (scratch_bytes < (int64_t)L.total) return PCB_EINVAL;
  int rc = pcb_bounded_draws(n, k, seed, labels, scratch, scratch_bytes, stream);
  if (rc != 0) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* base = (uint8_t*)scratch;
  int* counts = (int*)(base + L.off_counts);
  int* small = (int*)(base + L.off_small);
  cudaError_t e;
  // repeat { labels[hollow] = hollow } until no cluster is empty
  const int hgrid = (int)std::min<int64_t>((n + 255) / 256, 2L * sm_count());
  int passes = 0;
  while (true) {
    if ((e = cudaMemsetAsync(counts, 0, sizeof(int) * k, st)) != cudaSuccess) return (int)e;
    if ((e = cudaMemsetAsync(small + 1, 0, sizeof(int), st)) != cudaSuccess) return (int)e;
    if ((size_t)k * sizeof(int) <= 48 * 1024)
      init_hist_kernel<<<hgrid, 256, (size_t)k * sizeof(int), st>>>(labels, n, k, counts);
    else
      init_hist_global_kernel<<<hgrid, 256, 0, st>>>(labels, n, counts);
    PCB_CHECK_LAUNCH();
    init_fill_hollow<<<(k + 255) / 256, 256, 0, st>>>(counts, k, labels, small + 1);
    PCB_CHECK_LAUNCH();
    int flag = 0;
    if ((e = cudaMemcpyAsync(&flag, small + 1, sizeof(int), cudaMemcpyDeviceToHost, st)) != cudaSuccess)
      return (int)e;
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return (int)e;
    if (!flag) break;
    ++passes;
  }
  if (passes_out) *passes_out = passes;
  return 0;
}

// ---- synthesize_points (cli.py:102-105): Generator(PCG64(seed)).random((n, d)) ----
// numpy's random() = (next_uint64 >> 11) * 2^-53, one PCG64 output per value in
// row-major order; .astype(f32) rounds to nearest.
namespace pcb {
template <typename T>
__global__ void __launch_bounds__(256)
uniform_kernel(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t count, T* __restrict__ out) {
  const u128 state0 = ((u128)st_hi << 64) | st_lo, inc = ((u128)inc_hi << 64) | inc_lo;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t o0 = t * kOutPerThread;
  if (o0 >= count) return;
  u128 s = pcg_advance(state0, inc, (uint64_t)o0);
  const u128 M = pcg_mult();
  for (int q = 0; q < kOutPerThread && o0 + q < count; ++q) {
    s = s * M + inc;
    const double v = (double)(pcg_output(s) >> 11) * (1.0 / 9007199254740992.0);
    out[o0 + q] = (T)v;
  }
}
}  // namespace pcb

extern "C" int pcb_synthesize_uniform(int64_t count, uint64_t seed, int is_f64, void* out, void* stream) {
  if (count < 1 || !out) return PCB_EINVAL;
  u128 s0, inc;
  pcg64_from_seed(seed, &s0, &inc);
  const int64_t threads = (count + kOutPerThread - 1) / kOutPerThread;
  const unsigned grid = (unsigned)((threads + 255) / 256);
  cudaStream_t st = (cudaStream_t)stream;
  if (is_f64)
    uniform_kernel<double><<<grid, 256, 0, st>>>((uint64_t)(s0 >> 64), (uint64_t)s0, (uint64_t)(inc >> 64),
                                                 (uint64_t)inc, count, (double*)out);
  else
    uniform_kernel<float><<<grid, 256, 0, st>>>((uint64_t)(s0 >> 64), (uint64_t)s0, (uint64_t)(inc >> 64),
                                                (uint64_t)inc, count, (float*)out);
  PCB_CHECK_LAUNCH();
  return 0;
}
