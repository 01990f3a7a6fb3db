// Centroid update: per-cluster sums of point rows (clustering.py:282-288)
// and the own distances / objective of the new labels (clustering.py:148).
//
// The reference computes, for every cluster j, P[flatnonzero(labels==j)].mean(0)
// (k passes over the labels, f32 accumulation).  Here:
//   1. scan_counts:  exclusive scan of the cluster counts (already produced by
//                    the assignment kernel) -> segment offsets;
//   2. scatter:      counting sort of point ids by label; a warp aggregates
//                    equal labels with __match_any_sync so one atomic claims a
//                    run of slots per label and warp;
//   3. segment sums: a fixed partition of the sorted ids into slices; each
//                    slice walks its ids in order, gathering full point rows
//                    (coalesced, one row per warp step for large d) and
//                    accumulating in f64 registers; a label boundary flushes
//                    the partial with one RED.ADD.F64 per dimension.
// Every point row is read exactly once from HBM (n*d*sizeof(T) bytes), rows
// are contiguous, and no shared-memory atomics are needed (on sm_100 f32/f64
// shared atomics are CAS loops).  Sums are f64, so the f32 centroid
// sum/count is correctly rounded up to the ~1e-16 summation error.
#include "pcb_common.cuh"
#include "pcb_launch.cuh"

namespace pcb {

__global__ void __launch_bounds__(1024)
scan_counts(const double* __restrict__ counts, int k, int32_t* __restrict__ offsets,
            int32_t* __restrict__ cursor, const long long* __restrict__ state) {
  if (stopped(state) || delta_mode(state)) return;
  __shared__ int warp_tot[32];
  __shared__ int carry_s;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (int base = 0; base < k; base += blockDim.x) {
    const int j = base + threadIdx.x;
    const int c = j < k ? (int)counts[j] : 0;
    int x = c;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    if (w == 0) {
      int t = warp_tot[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      warp_tot[lane] = t;  // inclusive over warps
    }
    __syncthreads();
    const int carry = carry_s;
    const int excl = carry + (w > 0 ? warp_tot[w - 1] : 0) + x - c;
    if (j < k) { offsets[j] = excl; cursor[j] = excl; }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry_s = excl + c;
    __syncthreads();
  }
  if (threadIdx.x == 0) offsets[k] = carry_s;
}

__global__ void __launch_bounds__(256)
scatter_by_label(const int32_t* __restrict__ labels, int64_t n, int32_t* __restrict__ cursor,
                 int32_t* __restrict__ perm, const long long* __restrict__ state) {
  if (stopped(state) || delta_mode(state)) return;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const int64_t i = base + threadIdx.x;
    const bool live = i < n;
    const unsigned act = __ballot_sync(0xffffffffu, live);
    if (!live) continue;
    const int j = labels[i];
    const unsigned peers = __match_any_sync(act, j);
    const int leader = __ffs(peers) - 1;
    const int rank = __popc(peers & ((1u << lane) - 1u));
    int slot = 0;
    if (lane == leader) slot = atomicAdd(&cursor[j], __popc(peers));
    slot = __shfl_sync(peers, slot, leader);
    perm[slot + rank] = (int32_t)i;
  }
}

// Block-aggregated counting-sort scatter: a block ranks a chunk of ids per
// label in shared memory (native ATOMS.POPC.INC), claims one global range per
// (chunk, label), then writes.  ~k global atomics per 4096 ids instead of one
// per warp-label group.
constexpr int SC_EPT = 16;

__global__ void __launch_bounds__(256)
scatter_by_label_blocked(const int32_t* __restrict__ labels, int64_t n, int k, int32_t* __restrict__ cursor,
                         int32_t* __restrict__ perm, const long long* __restrict__ state) {
  if (stopped(state) || delta_mode(state)) return;
  extern __shared__ int sm[];
  int* hist = sm;
  int* base = sm + k;
  const int64_t chunk = (int64_t)blockDim.x * SC_EPT;
  const int64_t nchunks = (n + chunk - 1) / chunk;
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    for (int j = threadIdx.x; j < k; j += blockDim.x) hist[j] = 0;
    __syncthreads();
    int lab[SC_EPT], rnk[SC_EPT];
#pragma unroll
    for (int e = 0; e < SC_EPT; ++e) {
      const int64_t i = c * chunk + e * blockDim.x + threadIdx.x;
      lab[e] = i < n ? labels[i] : -1;
    }
#pragma unroll
    for (int e = 0; e < SC_EPT; ++e) rnk[e] = lab[e] >= 0 ? atomicAdd(&hist[lab[e]], 1) : 0;
    __syncthreads();
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
      const int h = hist[j];
      base[j] = h ? atomicAdd(&cursor[j], h) : 0;
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < SC_EPT; ++e) {
      const int64_t i = c * chunk + e * blockDim.x + threadIdx.x;
      if (lab[e] >= 0) perm[base[lab[e]] + rnk[e]] = (int32_t)i;
    }
    __syncthreads();
  }
}

// Largest j with offsets[j] <= s (segments may be empty: offsets non-decreasing).
__device__ __forceinline__ int segment_of(const int32_t* offsets, int k, int64_t s) {
  int lo = 0, hi = k - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (offsets[mid] <= s) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Exact own distance of a point to its centroid, in f64 from f32/f64 inputs:
// sum_t (p_t - c_t)^2.  This is what the objective sums (clustering.py:148),
// evaluated here — where the point row is already in registers — instead of
// in the assignment kernel, so every assignment variant (FFMA, 3xTF32 tensor
// cores) reports the same, correctly rounded own distances and objective.

// d > 16: one warp per slice of sorted ids; lane l owns dimensions l + 32 v.
template <typename T, int NV>
__global__ void __launch_bounds__(256)
segsum_warp(const T* __restrict__ P, int64_t n, int d, const int32_t* __restrict__ perm,
            const int32_t* __restrict__ offsets, int k, const T* __restrict__ C, int64_t slice,
            double* __restrict__ own_sorted, double* __restrict__ acc,
            const long long* __restrict__ state, int col0 = 0, int dw = -1, int pass = 3) {
  // Column slab [col0, col0 + dw) of every row (d > 1024 runs one launch per
  // slab of 1024 columns): pass bit 0 = first slab (own distances written),
  // bit 1 = last slab (own distances complete: objective).
  if (stopped(state) || delta_mode(state)) return;
  const AccLayout L{k, d};
  if (dw < 0) dw = d;
  P += col0;
  C += col0;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nslices = (n + slice - 1) / slice;
  double obj = 0.0;
  for (int64_t sl = warp; sl < nslices; sl += nwarps) {
    const int64_t s0 = sl * slice, s1 = min(n, s0 + slice);
    int j = segment_of(offsets, k, s0);
    int64_t jend = offsets[j + 1];
    double a[NV];
    T c[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int t = lane + 32 * v;
      a[v] = 0.0;
      c[v] = t < dw ? C[(int64_t)j * d + t] : T(0);
    }
    int64_t s = s0;
    while (s < s1) {
      if (s >= jend) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const int t = lane + 32 * v;
          if (t < dw) atomicAdd(&acc[(int64_t)j * d + col0 + t], a[v]);
          a[v] = 0.0;
        }
        do { ++j; jend = offsets[j + 1]; } while (s >= jend);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const int t = lane + 32 * v;
          c[v] = t < dw ? C[(int64_t)j * d + t] : T(0);
        }
      }
      const int64_t e = min(s1, jend);
      // two rows in flight per step
      for (; s + 2 <= e; s += 2) {
        const T* r0 = P + (int64_t)perm[s] * d;
        const T* r1 = P + (int64_t)perm[s + 1] * d;
        T x0[NV], x1[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const int t = lane + 32 * v;
          x0[v] = t < dw ? r0[t] : T(0);
          x1[v] = t < dw ? r1[t] : T(0);
        }
        double q0 = 0.0, q1 = 0.0;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          a[v] += (double)x0[v] + (double)x1[v];
          const double e0 = (double)x0[v] - (double)c[v], e1 = (double)x1[v] - (double)c[v];
          q0 = fma(e0, e0, q0);
          q1 = fma(e1, e1, q1);
        }
        q0 = warp_sum(q0);
        q1 = warp_sum(q1);
        if (lane == 0) {
          if (!(pass & 1)) { q0 += own_sorted[s]; q1 += own_sorted[s + 1]; }
          own_sorted[s] = q0;
          own_sorted[s + 1] = q1;
          if (pass & 2) obj += q0 + q1;
        }
      }
      if (s < e) {
        const T* r0 = P + (int64_t)perm[s] * d;
        double q0 = 0.0;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const int t = lane + 32 * v;
          const T x = t < dw ? r0[t] : T(0);
          a[v] += (double)x;
          const double e0 = (double)x - (double)c[v];
          q0 = fma(e0, e0, q0);
        }
        q0 = warp_sum(q0);
        if (lane == 0) {
          if (!(pass & 1)) q0 += own_sorted[s];
          own_sorted[s] = q0;
          if (pass & 2) obj += q0;
        }
        ++s;
      }
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int t = lane + 32 * v;
      if (t < dw) atomicAdd(&acc[(int64_t)j * d + col0 + t], a[v]);
    }
  }
  if (lane == 0 && obj != 0.0) atomicAdd(&acc[L.objective()], obj);
}

// f32 rows with d % 4 == 0 (64 < d <= 512): one warp per slice of sorted ids,
// lane l owns the float4 columns l + 32 v; four rows (16-byte loads, a whole
// 512-byte row per warp instruction at d = 128) are in flight per step.
template <int NV4>
__global__ void __launch_bounds__(256)
segsum_v4(const float* __restrict__ P, int64_t n, int d, const int32_t* __restrict__ perm,
          const int32_t* __restrict__ offsets, int k, const float* __restrict__ C, int64_t slice,
          double* __restrict__ own_sorted, double* __restrict__ acc, const long long* __restrict__ state) {
  if (stopped(state) || delta_mode(state)) return;
  const AccLayout L{k, d};
  const int lane = threadIdx.x & 31;
  const int d4 = d >> 2;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nslices = (n + slice - 1) / slice;
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  double obj = 0.0;
  for (int64_t sl = warp; sl < nslices; sl += nwarps) {
    const int64_t s0 = sl * slice, s1 = min(n, s0 + slice);
    int j = segment_of(offsets, k, s0);
    int64_t jend = offsets[j + 1];
    double a[NV4][4];
    float4 c[NV4];
#pragma unroll
    for (int v = 0; v < NV4; ++v) {
      const int f = lane + 32 * v;
      a[v][0] = a[v][1] = a[v][2] = a[v][3] = 0.0;
      c[v] = f < d4 ? reinterpret_cast<const float4*>(C + (int64_t)j * d)[f] : z4;
    }
    int64_t s = s0;
    while (s < s1) {
      if (s >= jend) {
#pragma unroll
        for (int v = 0; v < NV4; ++v) {
          const int f = lane + 32 * v;
          if (f < d4) {
            double* dst = acc + (int64_t)j * d + 4 * f;
            atomicAdd(dst + 0, a[v][0]);
            atomicAdd(dst + 1, a[v][1]);
            atomicAdd(dst + 2, a[v][2]);
            atomicAdd(dst + 3, a[v][3]);
          }
          a[v][0] = a[v][1] = a[v][2] = a[v][3] = 0.0;
        }
        do { ++j; jend = offsets[j + 1]; } while (s >= jend);
#pragma unroll
        for (int v = 0; v < NV4; ++v) {
          const int f = lane + 32 * v;
          c[v] = f < d4 ? reinterpret_cast<const float4*>(C + (int64_t)j * d)[f] : z4;
        }
      }
      const int64_t e = min(s1, jend);
      for (; s < e; s += 4) {
        const int nr = (int)(e - s < 4 ? e - s : 4);
        float4 x[4][NV4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const float4* row = reinterpret_cast<const float4*>(P + (int64_t)perm[r < nr ? s + r : s] * d);
#pragma unroll
          for (int v = 0; v < NV4; ++v) {
            const int f = lane + 32 * v;
            x[r][v] = (r < nr && f < d4) ? __ldcs(row + f) : z4;
          }
        }
        double q[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          q[r] = 0.0;
#pragma unroll
          for (int v = 0; v < NV4; ++v) {
            const float xs[4] = {x[r][v].x, x[r][v].y, x[r][v].z, x[r][v].w};
            const float cs[4] = {c[v].x, c[v].y, c[v].z, c[v].w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const double xd = (double)xs[i];
              a[v][i] += xd;
              const double ed = xd - (double)cs[i];
              q[r] = fma(ed, ed, q[r]);
            }
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
          for (int r = 0; r < 4; ++r) q[r] += __shfl_xor_sync(0xffffffffu, q[r], o);
        }
        if (lane < nr) {
          const double qo = lane == 0 ? q[0] : lane == 1 ? q[1] : lane == 2 ? q[2] : q[3];
          own_sorted[s + lane] = qo;
        }
        if (lane == 0) obj += q[0] + (nr > 1 ? q[1] : 0.0) + (nr > 2 ? q[2] : 0.0) + (nr > 3 ? q[3] : 0.0);
      }
      s = e;
    }
#pragma unroll
    for (int v = 0; v < NV4; ++v) {
      const int f = lane + 32 * v;
      if (f < d4) {
        double* dst = acc + (int64_t)j * d + 4 * f;
        atomicAdd(dst + 0, a[v][0]);
        atomicAdd(dst + 1, a[v][1]);
        atomicAdd(dst + 2, a[v][2]);
        atomicAdd(dst + 3, a[v][3]);
      }
    }
  }
  if (lane == 0 && obj != 0.0) atomicAdd(&acc[L.objective()], obj);
}

// d <= 16: one thread per slice, the whole row in registers.
template <typename T, int DP>
__global__ void __launch_bounds__(256)
segsum_thread(const T* __restrict__ P, int64_t n, int d, const int32_t* __restrict__ perm,
              const int32_t* __restrict__ offsets, int k, const T* __restrict__ C, int64_t slice,
              double* __restrict__ own_sorted, double* __restrict__ acc,
              const long long* __restrict__ state) {
  if (stopped(state) || delta_mode(state)) return;
  const AccLayout L{k, d};
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int64_t nslices = (n + slice - 1) / slice;
  double obj = 0.0;
  for (int64_t sl = tid; sl < nslices; sl += nth) {
    const int64_t s0 = sl * slice, s1 = min(n, s0 + slice);
    int j = segment_of(offsets, k, s0);
    int64_t jend = offsets[j + 1];
    double a[DP];
    T c[DP];
#pragma unroll
    for (int t = 0; t < DP; ++t) { a[t] = 0.0; c[t] = t < d ? C[(int64_t)j * d + t] : T(0); }
    for (int64_t s = s0; s < s1; ++s) {
      if (s >= jend) {
#pragma unroll
        for (int t = 0; t < DP; ++t) {
          if (t < d) atomicAdd(&acc[(int64_t)j * d + t], a[t]);
          a[t] = 0.0;
        }
        do { ++j; jend = offsets[j + 1]; } while (s >= jend);
#pragma unroll
        for (int t = 0; t < DP; ++t) c[t] = t < d ? C[(int64_t)j * d + t] : T(0);
      }
      const T* row = P + (int64_t)perm[s] * d;
      double q = 0.0;
#pragma unroll
      for (int t = 0; t < DP; ++t) {
        if (t < d) {
          const T x = row[t];
          a[t] += (double)x;
          const double e = (double)x - (double)c[t];
          q = fma(e, e, q);
        }
      }
      own_sorted[s] = q;
      obj += q;
    }
#pragma unroll
    for (int t = 0; t < DP; ++t)
      if (t < d) atomicAdd(&acc[(int64_t)j * d + t], a[t]);
  }
  obj = warp_sum(obj);
  if ((threadIdx.x & 31) == 0 && obj != 0.0) atomicAdd(&acc[L.objective()], obj);
}

template <typename T>
static int segment_sums(const T* P, int64_t n, int d, const int32_t* perm, const int32_t* offsets,
                        int k, const T* C, double* own, double* acc, const long long* state,
                        cudaStream_t st) {
  if (n < 1 || d < 1 || k < 1 || !P || !perm || !offsets || !acc || !C || !own) return PCB_EINVAL;
  const int sms = sm_count();
  if (d <= 16) {
    const int64_t threads = (int64_t)sms * 2048;
    int64_t slice = std::max<int64_t>(16, (n + threads - 1) / threads);
    const int64_t nsl = (n + slice - 1) / slice;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((nsl + 255) / 256, (int64_t)sms * 8));
#define PCB_SEG_T(DPV) segsum_thread<T, DPV><<<grid, 256, 0, st>>>(P, n, d, perm, offsets, k, C, slice, own, acc, state)
    if (d <= 2) PCB_SEG_T(2);
    else if (d <= 4) PCB_SEG_T(4);
    else if (d <= 8) PCB_SEG_T(8);
    else PCB_SEG_T(16);
#undef PCB_SEG_T
  } else {
    const int64_t warps = (int64_t)sms * 64;
    int64_t slice = std::max<int64_t>(64, (n + warps - 1) / warps);
    const int64_t nsl = (n + slice - 1) / slice;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((nsl * 32 + 255) / 256, (int64_t)sms * 8));
#define PCB_SEG_W(NVV) segsum_warp<T, NVV><<<grid, 256, 0, st>>>(P, n, d, perm, offsets, k, C, slice, own, acc, state)
#define PCB_SEG_V4(NV4) segsum_v4<NV4><<<grid, 256, 0, st>>>((const float*)P, n, d, perm, offsets, k, (const float*)C, slice, own, acc, state)
    if (sizeof(T) == 4 && d % 4 == 0 && d > 64 && d <= 512) {
      if (d <= 128) PCB_SEG_V4(1);
      else if (d <= 256) PCB_SEG_V4(2);
      else if (d <= 384) PCB_SEG_V4(3);
      else PCB_SEG_V4(4);
    }
    else if (d <= 32) PCB_SEG_W(1);
    else if (d <= 64) PCB_SEG_W(2);
    else if (d <= 128) PCB_SEG_W(4);
    else if (d <= 256) PCB_SEG_W(8);
    else if (d <= 512) PCB_SEG_W(16);
    else if (d <= 1024) PCB_SEG_W(32);
    else {
      // wider rows: slabs of 1024 columns, own distances accumulated across slabs
      for (int c0 = 0; c0 < d; c0 += 1024) {
        const int pass = (c0 == 0 ? 1 : 0) | (c0 + 1024 >= d ? 2 : 0);
        segsum_warp<T, 32><<<grid, 256, 0, st>>>(P, n, d, perm, offsets, k, C, slice, own, acc, state, c0,
                                                 std::min(1024, d - c0), pass);
        PCB_CHECK_LAUNCH();
      }
    }
#undef PCB_SEG_W
#undef PCB_SEG_V4
  }
  PCB_CHECK_LAUNCH();
  return 0;
}

// ---------------------------------------------------------------------------
// Delta centroid update.  Near convergence few labels change per iteration,
// so instead of re-summing every row the rank keeps its per-cluster f64 sums S
// (of its own rows, for the current labels) and adds/subtracts only the rows
// whose label changed.  The objective then follows from the sums exactly:
//   sum_i |p_i - c_l(i)|^2 = Q - 2 sum_j <c_j, S_j> + sum_j n_j |c_j|^2,
// Q = sum_i |p_i|^2 (f64, once per fit), c = the centroids the labels were
// assigned against (clustering.py:148 evaluates the same sum row by row).
// The full update (counting sort + segmented sums, exact own distances) runs
// whenever more than `frac` of the rows changed, a local cluster count is 0
// (the repair needs own distances), the sums are not valid yet, or a
// multi-rank repair moved points (state[kSumsStale]); it refreshes S.  The
// single-rank repair moves S in step with acc instead (repair.cu).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
update_mode_kernel(const double* __restrict__ acc, int k, int d, int64_t n, double frac, int force_full,
                   long long* __restrict__ state) {
  const AccLayout L{k, d};
  __shared__ int any_empty;
  if (threadIdx.x == 0) any_empty = 0;
  __syncthreads();
  for (int j = threadIdx.x; j < k; j += blockDim.x)
    if (acc[L.counts() + j] < 0.5) any_empty = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    const bool full = force_full || any_empty || state[kSumsStale] != 0 || acc[L.changed()] > frac * (double)n;
    // delta with the count pass's speculative changed-row sums already in S: 3
    // (a full update overwrites S from the full sums, discarding them)
    state[kMode] = full ? 0 : (state[kSpec] != 0 ? 3 : 1);
    state[kSumsStale] = 0;
    state[kSpec] = 0;
  }
}

// Changed rows only: S[new] += p, S[prev] -= p (f64), one warp per row.
template <typename T>
__global__ void __launch_bounds__(256)
delta_sums_kernel(const T* __restrict__ P, int64_t n, int d, const int32_t* __restrict__ prev,
                  const int32_t* __restrict__ labels, double* __restrict__ S, const long long* __restrict__ state) {
  if (stopped(state) || !delta_mode(state) || ((volatile const long long*)state)[kMode] == 3) return;
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // 4 groups of 32 labels in flight per warp and trip (the scan is a latency-
  // bound stream over 8 bytes per row; changed rows are ~0.1 % near convergence)
  for (int64_t base = w * 128; base < n; base += nw * 128) {
    int a[4], b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = base + 32 * u + lane;
      a[u] = i < n ? prev[i] : 0;
      b[u] = i < n ? labels[i] : 0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      unsigned m = __ballot_sync(0xffffffffu, a[u] != b[u]);
      while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        const int64_t r = base + 32 * u + src;
        const int ja = __shfl_sync(0xffffffffu, a[u], src), jb = __shfl_sync(0xffffffffu, b[u], src);
        for (int t = lane; t < d; t += 32) {
          const double x = (double)P[r * d + t];
          atomicAdd(&S[(int64_t)jb * d + t], x);
          atomicAdd(&S[(int64_t)ja * d + t], -x);
        }
      }
    }
  }
}

// Full mode: S <- the sums just computed.  Delta mode: acc sums <- S and the
// objective from the identity above.
template <typename T>
__global__ void __launch_bounds__(256)
delta_finish_kernel(const T* __restrict__ C, int k, int d, double* __restrict__ acc, double* __restrict__ S,
                    const double* __restrict__ Q, const long long* __restrict__ state) {
  if (stopped(state)) return;
  const AccLayout L{k, d};
  const int64_t kd = (int64_t)k * d;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  if (!delta_mode(state)) {
    for (int64_t e = tid; e < kd; e += nth) S[e] = acc[e];
    return;
  }
  double part = 0.0;
  for (int64_t e = tid; e < kd; e += nth) {
    const double s = S[e];
    acc[e] = s;
    const double c = (double)C[e];
    part += c * (acc[L.counts() + e / d] * c - 2.0 * s);
  }
  part = warp_sum(part);
  __shared__ double red[8];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) b += red[i];
    if (blockIdx.x == 0) b += *Q;
    atomicAdd(&acc[L.objective()], b);
  }
}

// sum of squares of all entries, f64 (Q of the objective identity)
template <typename T>
__global__ void __launch_bounds__(256)
sum_squares_kernel(const T* __restrict__ X, int64_t count, double* __restrict__ out) {
  double part = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
    const double x = (double)X[e];
    part = fma(x, x, part);
  }
  part = warp_sum(part);
  __shared__ double red[8];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) b += red[i];
    atomicAdd(out, b);
  }
}

}  // namespace pcb

extern "C" int pcb_sort_by_label(const int32_t* labels, int64_t n, int k, const double* counts,
                                 int32_t* offsets, int32_t* cursor, int32_t* perm,
                                 const long long* state, void* stream) {
  if (n < 1 || k < 1 || !labels || !counts || !offsets || !cursor || !perm) return PCB_EINVAL;
  if (n > INT32_MAX) return PCB_EUNSUP;
  cudaStream_t st = (cudaStream_t)stream;
  pcb::scan_counts<<<1, 1024, 0, st>>>(counts, k, offsets, cursor, state);
  PCB_CHECK_LAUNCH();
  const int sms = pcb::sm_count();
  if (k <= 6144) {
    const int64_t chunks = (n + 256 * pcb::SC_EPT - 1) / (256 * pcb::SC_EPT);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(chunks, (int64_t)sms * 4));
    pcb::scatter_by_label_blocked<<<grid, 256, 2 * k * sizeof(int), st>>>(labels, n, k, cursor, perm, state);
  } else {
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sms * 8));
    pcb::scatter_by_label<<<grid, 256, 0, st>>>(labels, n, cursor, perm, state);
  }
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_segment_sums_f32(const float* P, int64_t n, int d, const int32_t* perm,
                                    const int32_t* offsets, int k, const float* C, double* own_sorted,
                                    double* acc, const long long* state, void* stream) {
  return pcb::segment_sums<float>(P, n, d, perm, offsets, k, C, own_sorted, acc, state,
                                  (cudaStream_t)stream);
}

extern "C" int pcb_segment_sums_f64(const double* P, int64_t n, int d, const int32_t* perm,
                                    const int32_t* offsets, int k, const double* C, double* own_sorted,
                                    double* acc, const long long* state, void* stream) {
  return pcb::segment_sums<double>(P, n, d, perm, offsets, k, C, own_sorted, acc, state,
                                   (cudaStream_t)stream);
}

extern "C" int pcb_update_mode(const double* acc, int k, int d, int64_t n, double frac, int force_full,
                               long long* state, void* stream) {
  if (k < 1 || d < 1 || n < 1 || !acc || !state) return PCB_EINVAL;
  pcb::update_mode_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(acc, k, d, n, frac, force_full, state);
  PCB_CHECK_LAUNCH();
  return 0;
}

template <typename T>
static int delta_update(const T* P, int64_t n, int d, const int32_t* prev, const int32_t* labels, const T* C, int k,
                        double* S, const double* Q, double* acc, const long long* state, cudaStream_t st) {
  if (n < 1 || d < 1 || k < 1 || !P || !prev || !labels || !C || !S || !Q || !acc || !state) return PCB_EINVAL;
  const int sms = pcb::sm_count();
  // two blocks per SM (4 label groups in flight per warp): enough for the label
  // scan, and a cheap launch when the count pass already applied the sums (mode 3)
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sms * 2));
  pcb::delta_sums_kernel<T><<<grid, 256, 0, st>>>(P, n, d, prev, labels, S, state);
  PCB_CHECK_LAUNCH();
  const int64_t kd = (int64_t)k * d;
  const int g2 = (int)std::max<int64_t>(1, std::min<int64_t>((kd + 255) / 256, (int64_t)sms * 4));
  pcb::delta_finish_kernel<T><<<g2, 256, 0, st>>>(C, k, d, acc, S, Q, state);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_delta_update_f32(const float* P, int64_t n, int d, const int32_t* prev, const int32_t* labels,
                                    const float* C, int k, double* S, const double* Q, double* acc,
                                    const long long* state, void* stream) {
  return delta_update<float>(P, n, d, prev, labels, C, k, S, Q, acc, state, (cudaStream_t)stream);
}

extern "C" int pcb_delta_update_f64(const double* P, int64_t n, int d, const int32_t* prev, const int32_t* labels,
                                    const double* C, int k, double* S, const double* Q, double* acc,
                                    const long long* state, void* stream) {
  return delta_update<double>(P, n, d, prev, labels, C, k, S, Q, acc, state, (cudaStream_t)stream);
}

template <typename T>
static int sum_squares(const T* X, int64_t count, double* out, cudaStream_t st) {
  if (count < 1 || !X || !out) return PCB_EINVAL;
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), st);
  if (e != cudaSuccess) return (int)e;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((count + 255) / 256, (int64_t)pcb::sm_count() * 8));
  pcb::sum_squares_kernel<T><<<grid, 256, 0, st>>>(X, count, out);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_sum_squares_f32(const float* X, int64_t count, double* out, void* stream) {
  return sum_squares<float>(X, count, out, (cudaStream_t)stream);
}
extern "C" int pcb_sum_squares_f64(const double* X, int64_t count, double* out, void* stream) {
  return sum_squares<double>(X, count, out, (cudaStream_t)stream);
}
