// Host-side launch helpers shared by the kernel translation units.
#pragma once
#include <cuda_runtime.h>
#include <algorithm>
#include <stdint.h>

namespace pcb {

// SM count of the current device (cached per device).
int sm_count();

// Grid for a persistent kernel: SMs x resident blocks per SM.
template <typename K>
inline int persistent_grid(K kernel, int block, size_t smem) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  return per_sm * sm_count();
}

int assign_delta_f32(const float* P, const float* pnorm, int64_t n, int d, const float* C,
                     const float* cnorm, int k, const int32_t* labels_prev, int32_t* labels,
                     float* mind, double* acc, const long long* state, cudaStream_t st);

int assign_tc3xtf32_devcount(const float* phi, const float* plo, int ld, const float* pnorm, int64_t cap,
                             int d, const float* chi, const float* clo, const float* cnorm, int k,
                             int32_t* lab, const int* n_dev, const long long* state, cudaStream_t st,
                             const int* row_ids = nullptr, int* flag_list = nullptr, int* flag_count = nullptr);

// Exact argmin over all centroids of the rows flag_list[0 : *flag_count)
// (row r of P = P[row_ids[r]], or r); out[r] = label.  scratch:
// exact_scratch_bytes().
int exact_rows(const float* P, int d, const float* C, int k, const int* flag_list, const int* flag_count,
               const int* row_ids, int32_t* out, void* scratch, const long long* state, cudaStream_t st);
int64_t exact_scratch_bytes();

}  // namespace pcb
