// Shared device helpers for the B200 Lloyd hot path (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#include "../../include/popcorn_b200.h"

#if !defined(__CUDA_ARCH__) || __CUDA_ARCH__ >= 1000
#else
#error "popcorn_b200 targets sm_100a only"
#endif

namespace pcb {
// Host-side count of the kernels this library has launched (or recorded into
// a CUDA graph being captured); pcb_launch_count() reads it.
void count_launch();
}  // namespace pcb

// After every kernel launch: count it, then surface a launch error.
#define PCB_CHECK_LAUNCH() do { pcb::count_launch(); cudaError_t e__ = cudaGetLastError(); \
                                if (e__ != cudaSuccess) return (int)e__; } while (0)

namespace pcb {

constexpr int kWarp = 32;

// Layout of the fused per-iteration accumulator (f64), the buffer that is
// all-reduced across ranks: [ sums k*d | counts k | objective | changed ].
struct AccLayout {
  int64_t k, d;
  __host__ __device__ int64_t sums() const { return 0; }
  __host__ __device__ int64_t counts() const { return k * d; }
  __host__ __device__ int64_t objective() const { return k * d + k; }
  __host__ __device__ int64_t changed() const { return k * d + k + 1; }
  __host__ __device__ int64_t size() const { return k * d + k + 2; }
};

// Device loop state shared by all per-iteration kernels (int64 words):
//   [0] iterations recorded, [1] stop flag, [2] converged flag,
//   [3] repairs (moved points) of the current iteration,
//   [4] finalize block ticket, [5] non-finite distance seen,
//   [6] centroid-update mode of the iteration (0 full, 1 delta, 3 delta whose
//       changed-row sums the count pass already applied; update.cu),
//   [7] persistent per-cluster sums stale (a repair moved points),
//   [8] the count pass applied the changed-row sums speculatively (the
//       previous iteration was a delta one)
enum StateWord { kIters = 0, kStop = 1, kConverged = 2, kMoved = 3, kTicket = 4, kNanFlag = 5, kMode = 6,
                 kSumsStale = 7, kSpec = 8, kStateWords = 9 };

__device__ __forceinline__ bool stopped(const long long* state) {
  return state != nullptr && ((volatile const long long*)state)[kStop] != 0;
}

// Delta centroid update this iteration: the counting sort / segmented sums of
// the full update are skipped (they exit at once).
__device__ __forceinline__ bool delta_mode(const long long* state) {
  return state != nullptr && (((volatile const long long*)state)[kMode] & 1) != 0;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Order-preserving map float -> uint32 (total order; -0 < +0 is irrelevant here).
__device__ __forceinline__ uint32_t ordered_bits(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ uint64_t ordered_bits(double f) {
  unsigned long long u = (unsigned long long)__double_as_longlong(f);
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

// Argmin with lowest-index tie break (dense.py:56-68): (v, j) < (v', j') iff
// v < v' or (v == v' and j < j').
template <typename T>
__device__ __forceinline__ void argmin_merge(T& v, int& j, T v2, int j2) {
  if (v2 < v || (v2 == v && j2 < j)) { v = v2; j = j2; }
}

template <typename T>
__device__ __forceinline__ void warp_argmin(T& v, int& j) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T v2 = __shfl_xor_sync(0xffffffffu, v, o);
    int j2 = __shfl_xor_sync(0xffffffffu, j, o);
    argmin_merge(v, j, v2, j2);
  }
}

}  // namespace pcb
