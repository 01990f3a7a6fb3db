// One-time point preparation and the per-iteration finalize step.
//
//  * point norms            clustering.py:302   (accumulated in f64, rounded once)
//  * TF32 hi/lo split       operands of the 3xTF32 tensor-core kernel
//  * finalize               clustering.py:316 (_mean_centroids over the new
//                           labels, sums/counts from the all-reduced acc),
//                           cnorm for the next distance stage (clustering.py:310),
//                           history append + convergence test (clustering.py:319-324)
#include "pcb_common.cuh"
#include "pcb_launch.cuh"

namespace pcb {

template <typename T>
__global__ void __launch_bounds__(256)
point_norms_kernel(const T* __restrict__ P, int64_t n, int d, T* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  if (d >= 32) {  // warp per row
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = w; i < n; i += nw) {
      double s = 0.0;
      for (int t = lane; t < d; t += 32) { const double v = P[i * d + t]; s = fma(v, v, s); }
      s = warp_sum(s);
      if (lane == 0) out[i] = (T)s;
    }
  } else {        // thread per row
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
      double s = 0.0;
      for (int t = 0; t < d; ++t) { const double v = P[i * d + t]; s = fma(v, v, s); }
      out[i] = (T)s;
    }
  }
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__global__ void __launch_bounds__(256)
split_tf32_kernel(const float* __restrict__ X, int64_t rows, int d, int ld,
                  float* __restrict__ hi, float* __restrict__ lo) {
  const int64_t total = rows * (int64_t)ld;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / ld;
    const int t = (int)(e - r * ld);
    const float x = t < d ? X[r * d + t] : 0.0f;
    const float h = tf32_rna(x);
    hi[e] = h;
    lo[e] = x - h;  // exact in f32
  }
}

// One warp per centroid: c = sum / count (f64 divide, one rounding to T),
// cnorm accumulated in f64 from the rounded c, optional TF32 split.
// When `state` is non-null this is the per-iteration finalize: the last block
// to finish records history and evaluates convergence.
template <typename T>
__global__ void __launch_bounds__(256)
finalize_kernel(const double* __restrict__ acc, int k, int d, int64_t n_total,
                T* __restrict__ C, T* __restrict__ cnorm, float* __restrict__ c_hi,
                float* __restrict__ c_lo, int ld, double* __restrict__ obj_hist,
                long long* __restrict__ rep_hist, long long* __restrict__ state,
                int check_convergence, double tol) {
  if (stopped(state)) return;
  const AccLayout L{k, d};
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = w; j < k; j += nw) {
    const double cnt = acc[L.counts() + j];
    double s2 = 0.0;
    for (int t = lane; t < d; t += 32) {
      const T c = cnt > 0.0 ? (T)(acc[j * d + t] / cnt) : T(0);
      C[j * d + t] = c;
      s2 = fma((double)c, (double)c, s2);
    }
    if (c_hi != nullptr) {
      for (int t = lane; t < ld; t += 32) {
        const float x = t < d ? (float)C[j * d + t] : 0.0f;
        const float h = tf32_rna(x);
        c_hi[j * ld + t] = h;
        c_lo[j * ld + t] = x - h;
      }
    }
    s2 = warp_sum(s2);
    if (lane == 0) cnorm[j] = (T)s2;
  }
  if (state == nullptr) return;
  // last-block-done: record history, convergence test (clustering.py:319-324)
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long t = atomicAdd((unsigned long long*)&state[kTicket], 1ull);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence();
  state[kTicket] = 0;
  const long long it = state[kIters];
  obj_hist[it] = acc[L.objective()];
  rep_hist[it] = state[kMoved];
  state[kMoved] = 0;
  state[kIters] = it + 1;
  const double changed = acc[L.changed()] / (double)n_total;
  if (check_convergence && changed <= tol) {
    state[kConverged] = 1;
    state[kStop] = 1;
  }
}

template <typename T>
__global__ void __launch_bounds__(256)
centroid_norms_kernel(const T* __restrict__ C, int k, int d, T* __restrict__ cnorm,
                      float* __restrict__ c_hi, float* __restrict__ c_lo, int ld) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = w; j < k; j += nw) {
    double s2 = 0.0;
    for (int t = lane; t < d; t += 32) { const double c = C[j * d + t]; s2 = fma(c, c, s2); }
    if (c_hi != nullptr) {
      for (int t = lane; t < ld; t += 32) {
        const float x = t < d ? (float)C[j * d + t] : 0.0f;
        const float h = tf32_rna(x);
        c_hi[j * ld + t] = h;
        c_lo[j * ld + t] = x - h;
      }
    }
    s2 = warp_sum(s2);
    if (lane == 0) cnorm[j] = (T)s2;
  }
}

static inline int blocks_for(int64_t work, int per_block) {
  const int64_t b = (work + per_block - 1) / per_block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)sm_count() * 16));
}

template <typename T>
static int finalize(const double* acc, int k, int d, int64_t n_total, T* C, T* cnorm, float* hi,
                    float* lo, int ld, double* oh, long long* rh, long long* state, int cc,
                    double tol, cudaStream_t st) {
  if (k < 1 || d < 1 || !acc || !C || !cnorm) return PCB_EINVAL;
  if (state && (!oh || !rh)) return PCB_EINVAL;
  if (hi && (!lo || ld < d)) return PCB_EINVAL;
  finalize_kernel<T><<<blocks_for(k, 8), 256, 0, st>>>(acc, k, d, n_total, C, cnorm, hi, lo, ld,
                                                         oh, rh, state, cc, tol);
  PCB_CHECK_LAUNCH();
  return 0;
}

}  // namespace pcb

using namespace pcb;

extern "C" int pcb_point_norms_f32(const float* P, int64_t n, int d, float* pnorm, void* stream) {
  if (n < 1 || d < 1 || !P || !pnorm) return PCB_EINVAL;
  point_norms_kernel<float><<<blocks_for(d >= 32 ? n * 32 : n, 256), 256, 0, (cudaStream_t)stream>>>(P, n, d, pnorm);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_point_norms_f64(const double* P, int64_t n, int d, double* pnorm, void* stream) {
  if (n < 1 || d < 1 || !P || !pnorm) return PCB_EINVAL;
  point_norms_kernel<double><<<blocks_for(d >= 32 ? n * 32 : n, 256), 256, 0, (cudaStream_t)stream>>>(P, n, d, pnorm);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_split_tf32(const float* X, int64_t rows, int d, int ld, float* hi, float* lo,
                              void* stream) {
  if (rows < 1 || d < 1 || ld < d || !X || !hi || !lo) return PCB_EINVAL;
  split_tf32_kernel<<<blocks_for(rows * ld, 256), 256, 0, (cudaStream_t)stream>>>(X, rows, d, ld, hi, lo);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_finalize_f32(const double* acc, int k, int d, int64_t n_total, float* C,
                                float* cnorm, float* c_hi, float* c_lo, int ld,
                                double* objective_hist, long long* repairs_hist, long long* state,
                                int check_convergence, double tol, void* stream) {
  return finalize<float>(acc, k, d, n_total, C, cnorm, c_hi, c_lo, ld, objective_hist,
                         repairs_hist, state, check_convergence, tol, (cudaStream_t)stream);
}

extern "C" int pcb_finalize_f64(const double* acc, int k, int d, int64_t n_total, double* C,
                                double* cnorm, double* objective_hist, long long* repairs_hist,
                                long long* state, int check_convergence, double tol, void* stream) {
  return finalize<double>(acc, k, d, n_total, C, cnorm, nullptr, nullptr, 0, objective_hist,
                          repairs_hist, state, check_convergence, tol, (cudaStream_t)stream);
}

extern "C" int pcb_centroids_from_acc_f32(const double* acc, int k, int d, float* C, float* cnorm,
                                          float* c_hi, float* c_lo, int ld, void* stream) {
  return finalize<float>(acc, k, d, 1, C, cnorm, c_hi, c_lo, ld, nullptr, nullptr, nullptr, 0, 0.0,
                         (cudaStream_t)stream);
}

extern "C" int pcb_centroids_from_acc_f64(const double* acc, int k, int d, double* C,
                                          double* cnorm, void* stream) {
  return finalize<double>(acc, k, d, 1, C, cnorm, nullptr, nullptr, 0, nullptr, nullptr, nullptr, 0,
                          0.0, (cudaStream_t)stream);
}

extern "C" int pcb_centroid_norms_f32(const float* C, int k, int d, float* cnorm, float* c_hi,
                                      float* c_lo, int ld, void* stream) {
  if (k < 1 || d < 1 || !C || !cnorm || (c_hi && (!c_lo || ld < d))) return PCB_EINVAL;
  centroid_norms_kernel<float><<<blocks_for(k, 8), 256, 0, (cudaStream_t)stream>>>(C, k, d, cnorm, c_hi, c_lo, ld);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_centroid_norms_f64(const double* C, int k, int d, double* cnorm, void* stream) {
  if (k < 1 || d < 1 || !C || !cnorm) return PCB_EINVAL;
  centroid_norms_kernel<double><<<blocks_for(k, 8), 256, 0, (cudaStream_t)stream>>>(C, k, d, cnorm, nullptr, nullptr, 0);
  PCB_CHECK_LAUNCH();
  return 0;
}

// Input validation on the device (validation.py:45-46 semantics): number of
// non-finite entries of X, so the driver can raise ValueError without a host
// pass over n*d values.
template <typename T>
__global__ void __launch_bounds__(256)
count_nonfinite_kernel(const T* __restrict__ X, int64_t count, unsigned long long* __restrict__ out) {
  unsigned long long c = 0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x)
    c += !isfinite(X[e]);
  c = pcb::warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

extern "C" int pcb_count_nonfinite_f32(const float* X, int64_t count, unsigned long long* out, void* stream) {
  if (count < 0 || !X || !out) return PCB_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return (int)e;
  count_nonfinite_kernel<float><<<blocks_for(count, 1024), 256, 0, st>>>(X, count, out);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_count_nonfinite_f64(const double* X, int64_t count, unsigned long long* out, void* stream) {
  if (count < 0 || !X || !out) return PCB_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return (int)e;
  count_nonfinite_kernel<double><<<blocks_for(count, 1024), 256, 0, st>>>(X, count, out);
  PCB_CHECK_LAUNCH();
  return 0;
}
