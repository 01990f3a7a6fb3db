// Empty-cluster repair on the device (clustering.py:111-139, called from
// _assignment_step clustering.py:146).
//
// Semantics reproduced exactly: while some cluster is empty, for each cluster
// that was empty at the start of the pass, in ascending order, the point with
// the largest own distance D[i, label_i] among points not moved yet (ties ->
// lowest index) is moved to that cluster.  Own distances of unmoved points
// never change (their labels do not), so mind[] from the assignment kernel is
// the reference's `own` vector; a moved point gets mind = -inf.
//
// One cooperative launch (grid = SMs x occupancy) does the whole thing with a
// grid-wide argmax per donor (one grid.sync per donor: block keys are double
// buffered and every block reduces them redundantly).  When no cluster is
// empty — the common case — every block sees that from the counts and exits
// before any grid barrier.  The fused accumulator is patched in place
// (sums, counts, objective, changed) so the update and finalize kernels see
// the post-repair state; state[kMoved] counts the donations
// (ClusteringResult.repairs).
#include <cooperative_groups.h>

#include "pcb_common.cuh"
#include "pcb_launch.cuh"

namespace cg = cooperative_groups;

namespace pcb {

struct DonorKey {
  double v;
  long long i;
};

__device__ __forceinline__ void argmax_merge(DonorKey& a, const DonorKey& b) {
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) a = b;
}

template <typename T>
__device__ double pair_distance(const T* P, const T* pnorm, const T* C, const T* cnorm, int d,
                                int64_t i, int j) {
  // same association as the assignment kernels: pnorm + (cnorm - 2<p,c>)
  T dot = T(0);
  for (int t = 0; t < d; ++t) dot = fma(P[i * d + t], C[(int64_t)j * d + t], dot);
  const T s = fma(T(-2), dot, cnorm[j]);
  return (double)(pnorm[i] + s);
}

template <typename T>
__global__ void __launch_bounds__(256)
repair_kernel(const T* __restrict__ P, const T* __restrict__ pnorm, int64_t n, int d,
              const T* __restrict__ C, const T* __restrict__ cnorm, int k,
              const int32_t* __restrict__ labels_prev, int32_t* __restrict__ labels,
              T* __restrict__ mind, double* __restrict__ acc, long long* __restrict__ state,
              DonorKey* __restrict__ keys /* 2*gridDim */, int* __restrict__ elist /* k+1 */) {
  if (stopped(state)) return;
  cg::grid_group grid = cg::this_grid();
  const AccLayout L{k, d};
  __shared__ int s_any;
  __shared__ DonorKey s_warp[8];
  if (threadIdx.x == 0) s_any = 0;
  __syncthreads();
  for (int j = threadIdx.x; j < k; j += blockDim.x)
    if (acc[L.counts() + j] == 0.0) s_any = 1;
  __syncthreads();
  if (!s_any) return;  // identical decision in every block: no barrier reached

  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = (int64_t)blockIdx.x * per, hi = min(n, lo + per);
  int parity = 0;
  while (true) {
    grid.sync();  // counts of the previous pass are final
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      int c = 0;
      for (int j = 0; j < k; ++j)
        if (acc[L.counts() + j] == 0.0) elist[1 + c++] = j;
      elist[0] = c;
    }
    grid.sync();
    const int ne = ((volatile int*)elist)[0];
    if (ne == 0) break;
    for (int e = 0; e < ne; ++e) {
      const int j = ((volatile int*)elist)[1 + e];
      // block-local argmax of own distance over unmoved points
      DonorKey best{-INFINITY, n};
      for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        DonorKey c{(double)mind[i], i};
        argmax_merge(best, c);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        DonorKey b{__shfl_xor_sync(0xffffffffu, best.v, o), __shfl_xor_sync(0xffffffffu, best.i, o)};
        argmax_merge(best, b);
      }
      if ((threadIdx.x & 31) == 0) s_warp[threadIdx.x >> 5] = best;
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) argmax_merge(best, s_warp[w]);
        keys[parity * gridDim.x + blockIdx.x] = best;
      }
      __syncthreads();
      grid.sync();
      // every block reduces the block keys redundantly; the block whose slice
      // holds the donor applies the donation, so its own next scan already
      // sees mind[donor] = -inf without another grid barrier.
      if (threadIdx.x < 32) {
        DonorKey g{-INFINITY, n};
        for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) argmax_merge(g, keys[parity * gridDim.x + b]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          DonorKey b{__shfl_xor_sync(0xffffffffu, g.v, o), __shfl_xor_sync(0xffffffffu, g.i, o)};
          argmax_merge(g, b);
        }
        const int64_t donor = g.i;
        if (donor >= lo && donor < hi) {
          const int old = labels[donor];
          for (int t = threadIdx.x; t < d; t += 32) {
            const double p = (double)P[donor * d + t];
            atomicAdd(&acc[(int64_t)old * d + t], -p);
            atomicAdd(&acc[(int64_t)j * d + t], p);
          }
          if (threadIdx.x == 0) {
            const double dnew = pair_distance(P, pnorm, C, cnorm, d, donor, j);
            atomicAdd(&acc[L.objective()], dnew - (double)mind[donor]);
            if (labels_prev != nullptr) {
              const int prev = labels_prev[donor];
              atomicAdd(&acc[L.changed()], (double)((j != prev) - (old != prev)));
            }
            atomicAdd(&acc[L.counts() + old], -1.0);
            atomicAdd(&acc[L.counts() + j], 1.0);
            labels[donor] = j;
            mind[donor] = T(-INFINITY);
            atomicAdd((unsigned long long*)&state[kMoved], 1ull);
          }
        }
      }
      __syncthreads();
      parity ^= 1;
    }
  }
}

// Cooperative grid: one block per SM (the argmax is L2-bound; more blocks
// only add barrier cost).
static int repair_grid() { return sm_count(); }

static size_t repair_scratch(int k) {
  return sizeof(DonorKey) * 2 * (size_t)repair_grid() + sizeof(int) * (size_t)(k + 1);
}

template <typename T>
static int repair(const T* P, const T* pnorm, int64_t n, int d, const T* C, const T* cnorm, int k,
                  const int32_t* lp, int32_t* lab, T* mind, double* acc, long long* state,
                  void* scratch, int64_t scratch_bytes, cudaStream_t st) {
  if (n < 1 || d < 1 || k < 1 || !P || !pnorm || !C || !cnorm || !lab || !mind || !acc || !state ||
      !scratch)
    return PCB_EINVAL;
  if (scratch_bytes < (int64_t)repair_scratch(k)) return PCB_EINVAL;
  auto kern = repair_kernel<T>;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
  if (e != cudaSuccess) return (int)e;
  if (per_sm < 1) return PCB_EUNSUP;
  const int grid = repair_grid();
  DonorKey* keys = (DonorKey*)scratch;
  int* elist = (int*)(keys + 2 * grid);
  void* args[] = {(void*)&P, (void*)&pnorm, (void*)&n, (void*)&d, (void*)&C, (void*)&cnorm,
                  (void*)&k, (void*)&lp, (void*)&lab, (void*)&mind, (void*)&acc, (void*)&state,
                  (void*)&keys, (void*)&elist};
  e = cudaLaunchCooperativeKernel((void*)kern, dim3(grid), dim3(256), args, 0, st);
  return (int)e;
}

}  // namespace pcb

extern "C" int64_t pcb_repair_scratch_bytes(int k) { return (int64_t)pcb::repair_scratch(k); }

extern "C" int pcb_repair_f32(const float* P, const float* pnorm, int64_t n, int d, const float* C,
                              const float* cnorm, int k, const int32_t* labels_prev, int32_t* labels,
                              float* mind, double* acc, long long* state, void* scratch,
                              int64_t scratch_bytes, void* stream) {
  return pcb::repair<float>(P, pnorm, n, d, C, cnorm, k, labels_prev, labels, mind, acc, state,
                            scratch, scratch_bytes, (cudaStream_t)stream);
}

extern "C" int pcb_repair_f64(const double* P, const double* pnorm, int64_t n, int d,
                              const double* C, const double* cnorm, int k,
                              const int32_t* labels_prev, int32_t* labels, double* mind,
                              double* acc, long long* state, void* scratch, int64_t scratch_bytes,
                              void* stream) {
  return pcb::repair<double>(P, pnorm, n, d, C, cnorm, k, labels_prev, labels, mind, acc, state,
                             scratch, scratch_bytes, (cudaStream_t)stream);
}

// ---------------------------------------------------------------------------
// Multi-rank repair building blocks (host-orchestrated, rare path).  The
// driver all-gathers the per-rank argmax keys, the owner rank applies the
// donation locally and publishes a delta record that every rank commits to
// its (already all-reduced, hence identical) accumulator.
//   delta layout (f64, d+4 words): [ p_donor (d) | old label | d_objective |
//                                    d_changed | valid ]
// ---------------------------------------------------------------------------
namespace pcb {

template <typename T>
__global__ void __launch_bounds__(1024)
argmax_own_kernel(const T* __restrict__ mind, int64_t n, int64_t offset, double* __restrict__ out) {
  __shared__ DonorKey s_warp[32];
  DonorKey best{-INFINITY, offset + n};
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    DonorKey c{(double)mind[i], offset + i};
    argmax_merge(best, c);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    DonorKey b{__shfl_xor_sync(0xffffffffu, best.v, o), __shfl_xor_sync(0xffffffffu, best.i, o)};
    argmax_merge(best, b);
  }
  if ((threadIdx.x & 31) == 0) s_warp[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) argmax_merge(best, s_warp[w]);
    out[0] = best.v;
    out[1] = (double)best.i;
  }
}

template <typename T>
__global__ void repair_apply_kernel(const T* __restrict__ P, const T* __restrict__ pnorm, int d,
                                    const T* __restrict__ C, const T* __restrict__ cnorm,
                                    const int32_t* __restrict__ labels_prev,
                                    int32_t* __restrict__ labels, T* __restrict__ mind,
                                    int64_t donor, int j, double* __restrict__ delta) {
  for (int t = threadIdx.x; t < d; t += blockDim.x) delta[t] = (double)P[donor * d + t];
  if (threadIdx.x == 0) {
    const int old = labels[donor];
    const double dnew = pair_distance(P, pnorm, C, cnorm, d, donor, j);
    delta[d] = (double)old;
    delta[d + 1] = dnew - (double)mind[donor];
    delta[d + 2] = labels_prev ? (double)((j != labels_prev[donor]) - (old != labels_prev[donor])) : 0.0;
    delta[d + 3] = 1.0;
    labels[donor] = j;
    mind[donor] = T(-INFINITY);
  }
}

__global__ void repair_commit_kernel(double* __restrict__ acc, int k, int d, int j,
                                     const double* __restrict__ delta, long long* __restrict__ state) {
  const AccLayout L{k, d};
  if (delta[d + 3] != 1.0) return;
  const int old = (int)delta[d];
  for (int t = threadIdx.x; t < d; t += blockDim.x) {
    acc[(int64_t)old * d + t] -= delta[t];
    acc[(int64_t)j * d + t] += delta[t];
  }
  if (threadIdx.x == 0) {
    acc[L.counts() + old] -= 1.0;
    acc[L.counts() + j] += 1.0;
    acc[L.objective()] += delta[d + 1];
    acc[L.changed()] += delta[d + 2];
    state[kMoved] += 1;
  }
}

}  // namespace pcb

extern "C" int pcb_argmax_own_f32(const float* mind, int64_t n, int64_t offset, double* out2,
                                  void* stream) {
  if (n < 1 || !mind || !out2) return PCB_EINVAL;
  pcb::argmax_own_kernel<float><<<1, 1024, 0, (cudaStream_t)stream>>>(mind, n, offset, out2);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_argmax_own_f64(const double* mind, int64_t n, int64_t offset, double* out2,
                                  void* stream) {
  if (n < 1 || !mind || !out2) return PCB_EINVAL;
  pcb::argmax_own_kernel<double><<<1, 1024, 0, (cudaStream_t)stream>>>(mind, n, offset, out2);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_repair_apply_f32(const float* P, const float* pnorm, int d, const float* C,
                                    const float* cnorm, const int32_t* labels_prev,
                                    int32_t* labels, float* mind, int64_t donor_local, int j,
                                    double* delta, void* stream) {
  if (d < 1 || !P || !labels || !mind || !delta || donor_local < 0) return PCB_EINVAL;
  pcb::repair_apply_kernel<float><<<1, 128, 0, (cudaStream_t)stream>>>(
      P, pnorm, d, C, cnorm, labels_prev, labels, mind, donor_local, j, delta);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_repair_apply_f64(const double* P, const double* pnorm, int d, const double* C,
                                    const double* cnorm, const int32_t* labels_prev,
                                    int32_t* labels, double* mind, int64_t donor_local, int j,
                                    double* delta, void* stream) {
  if (d < 1 || !P || !labels || !mind || !delta || donor_local < 0) return PCB_EINVAL;
  pcb::repair_apply_kernel<double><<<1, 128, 0, (cudaStream_t)stream>>>(
      P, pnorm, d, C, cnorm, labels_prev, labels, mind, donor_local, j, delta);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_repair_commit(double* acc, int k, int d, int j, const double* delta,
                                 long long* state, void* stream) {
  if (k < 1 || d < 1 || !acc || !delta || !state) return PCB_EINVAL;
  pcb::repair_commit_kernel<<<1, 128, 0, (cudaStream_t)stream>>>(acc, k, d, j, delta, state);
  PCB_CHECK_LAUNCH();
  return 0;
}
