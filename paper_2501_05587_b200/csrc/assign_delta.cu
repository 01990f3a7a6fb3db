// delta-chunked P.C.P^T distance stage — the ablation of PAPER.md:146-237.
//
// The related-document attachment writes the squared distance of point p to
// centroid c as the bilinear form q C q^T with q = [1, p] and the augmented
// (d+1) x (d+1) matrix C = [[|c|^2, -c^T], [-c, I]] (analysis.py:83-102), pads
// r = d+1 to a multiple of delta, splits C and P into delta x delta blocks and
// forms D_i = P_i C P_i^T per row chunk, keeping only the diagonal and skipping
// the blocks C_ab = 0 (a, b > 1, a != b).  Per centroid the
// non-zero blocks are: the first block column C_a1 (first column -c), the first
// block row C_1b (first row -c) and the diagonal blocks C_bb (identity; the
// corner block also holds |c|^2).  This kernel evaluates exactly that block
// algebra, materialising every non-zero delta x delta block in shared memory
// and multiplying it as a dense block (the scheme's cost model: ~3 r delta
// MACs per point-centroid pair instead of d for the fused GEMM):
//
//   T_1 = sum_a q_a C_a1,   T_b = q_1 C_1b + q_b C_bb (b > 1),
//   D   = T_1 . q_1 + sum_{b>1} T_b . q_b
//
// SIMT FP32, 32 points x 32 centroids per block, each thread 2 x 2 pairs.
// It is kept as an ablation against the fused tensor-core kernels; the
// bookkeeping (labels, counts, changed) matches the other assignment kernels.
#include "pcb_common.cuh"
#include "pcb_launch.cuh"

namespace pcb {

constexpr int DL = 8;          // delta
constexpr int DBP = 32;        // points per block
constexpr int DBC = 32;        // centroids per block tile

// q-block b of point i: q = [1, p_1..p_d, 0...]
__device__ __forceinline__ float qval(const float* __restrict__ P, int64_t i, int d, int t) {
  return t == 0 ? 1.0f : (t <= d ? P[i * d + (t - 1)] : 0.0f);
}

// entry (u, v) of block (a, b) of C_j, a/b block indices, augmented indexing
__device__ __forceinline__ float cval(const float* __restrict__ C, const float* __restrict__ cn, int j, int d,
                                      int a, int b, int u, int v) {
  const int r = a * DL + u, c = b * DL + v;
  if (r == 0 && c == 0) return cn[j];
  if (r == 0) return c <= d ? -C[(int64_t)j * d + (c - 1)] : 0.0f;
  if (c == 0) return r <= d ? -C[(int64_t)j * d + (r - 1)] : 0.0f;
  return (r == c && r <= d) ? 1.0f : 0.0f;
}

__global__ void __launch_bounds__(256)
assign_delta_kernel(const float* __restrict__ P, const float* __restrict__ pnorm, int64_t n, int d,
                    const float* __restrict__ C, const float* __restrict__ cnorm, int k,
                    const int32_t* __restrict__ labels_prev, int32_t* __restrict__ labels,
                    float* __restrict__ mind, double* __restrict__ acc, const long long* __restrict__ state) {
  if (stopped(state)) return;
  __shared__ float q1[DBP][DL];           // first q block of each point
  __shared__ float qb[DBP][DL];           // current q block
  __shared__ float Cb1[DBC][DL][DL + 1];  // C_b1 of each centroid (block column 1)
  __shared__ float C1b[DBC][DL][DL + 1];  // C_1b (block row 1)
  __shared__ float Cbb[DBC][DL][DL + 1];  // C_bb (diagonal block)
  __shared__ float bestv[DBP][16];
  __shared__ int bestj[DBP][16];
  __shared__ int hist_s[2048];
  const AccLayout L{k, d};
  const int nblk = (d + 1 + DL - 1) / DL;  // Delta r
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, 2 x 2 pairs each
  const bool use_hist = acc != nullptr && k <= 2048;
  if (use_hist)
    for (int j = threadIdx.x; j < k; j += blockDim.x) hist_s[j] = 0;
  long long chg = 0;
  const int64_t ptiles = (n + DBP - 1) / DBP;
  for (int64_t pt = blockIdx.x; pt < ptiles; pt += gridDim.x) {
    const int64_t p0 = pt * DBP;
    float bv[2] = {INFINITY, INFINITY};
    int bj[2] = {0, 0};
    __syncthreads();
    for (int e = threadIdx.x; e < DBP * DL; e += blockDim.x) {
      const int pi = e / DL, u = e % DL;
      const int64_t i = min(p0 + pi, n - 1);
      q1[pi][u] = qval(P, i, d, u);
    }
    for (int c0 = 0; c0 < k; c0 += DBC) {
      float T1[2][2][DL];
      float D[2][2];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          D[a][c] = 0.0f;
#pragma unroll
          for (int v = 0; v < DL; ++v) T1[a][c][v] = 0.0f;
        }
      for (int b = 0; b < nblk; ++b) {
        __syncthreads();
        for (int e = threadIdx.x; e < DBP * DL; e += blockDim.x) {
          const int pi = e / DL, u = e % DL;
          const int64_t i = min(p0 + pi, n - 1);
          qb[pi][u] = qval(P, i, d, b * DL + u);
        }
        for (int e = threadIdx.x; e < DBC * DL * DL; e += blockDim.x) {
          const int cj = e / (DL * DL), u = (e / DL) % DL, v = e % DL;
          const int j = min(c0 + cj, k - 1);
          Cb1[cj][u][v] = cval(C, cnorm, j, d, b, 0, u, v);
          C1b[cj][u][v] = b > 0 ? cval(C, cnorm, j, d, 0, b, u, v) : 0.0f;
          Cbb[cj][u][v] = b > 0 ? cval(C, cnorm, j, d, b, b, u, v) : 0.0f;
        }
        __syncthreads();
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          const int pi = ty + 16 * a;
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int cj = tx + 16 * c;
            // T_1 += q_b C_b1 (dense delta x delta block product)
#pragma unroll
            for (int u = 0; u < DL; ++u) {
              const float qu = qb[pi][u];
#pragma unroll
              for (int v = 0; v < DL; ++v) T1[a][c][v] = fmaf(qu, Cb1[cj][u][v], T1[a][c][v]);
            }
            if (b > 0) {
              // T_b = q_1 C_1b + q_b C_bb ; D += T_b . q_b
#pragma unroll
              for (int v = 0; v < DL; ++v) {
                float tb = 0.0f;
#pragma unroll
                for (int u = 0; u < DL; ++u) tb = fmaf(q1[pi][u], C1b[cj][u][v], tb);
#pragma unroll
                for (int u = 0; u < DL; ++u) tb = fmaf(qb[pi][u], Cbb[cj][u][v], tb);
                D[a][c] = fmaf(tb, qb[pi][v], D[a][c]);
              }
            }
          }
        }
      }
      // D += T_1 . q_1, then the running argmin (ascending centroid index)
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        const int pi = ty + 16 * a;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          float dd = D[a][c];
#pragma unroll
          for (int v = 0; v < DL; ++v) dd = fmaf(T1[a][c][v], q1[pi][v], dd);
          const int j = c0 + tx + 16 * c;
          if (j < k) argmin_merge(bv[a], bj[a], dd, j);
        }
      }
    }
    // merge over the 16 threads sharing each point
    __syncthreads();
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      bestv[ty + 16 * a][tx] = bv[a];
      bestj[ty + 16 * a][tx] = bj[a];
    }
    __syncthreads();
    if (threadIdx.x < DBP) {
      const int pi = threadIdx.x;
      float v = bestv[pi][0];
      int j = bestj[pi][0];
      for (int t = 1; t < 16; ++t) argmin_merge(v, j, bestv[pi][t], bestj[pi][t]);
      const int64_t i = p0 + pi;
      if (i < n) {
        labels[i] = j;
        if (mind) mind[i] = v;
        if (acc) {
          if (labels_prev) chg += (labels_prev[i] != j);
          if (use_hist) atomicAdd(&hist_s[j], 1);
          else atomicAdd(&acc[L.counts() + j], 1.0);
        }
        if (state != nullptr && !isfinite(v)) atomicExch((unsigned long long*)&state[kNanFlag], 1ull);
      }
    }
  }
  if (acc) {
    if (threadIdx.x < 32) {
      chg = warp_sum(chg);
      if (threadIdx.x == 0 && chg) atomicAdd(&acc[L.changed()], (double)chg);
    }
    __syncthreads();
    if (use_hist)
      for (int j = threadIdx.x; j < k; j += blockDim.x)
        if (hist_s[j]) atomicAdd(&acc[L.counts() + j], (double)hist_s[j]);
  }
}

int assign_delta_f32(const float* P, const float* pnorm, int64_t n, int d, const float* C, const float* cnorm,
                     int k, const int32_t* labels_prev, int32_t* labels, float* mind, double* acc,
                     const long long* state, cudaStream_t st) {
  if (n < 1 || d < 1 || k < 1 || !P || !C || !cnorm || !labels) return PCB_EINVAL;
  const int64_t tiles = (n + DBP - 1) / DBP;
  const int grid = (int)std::min<int64_t>(tiles, (int64_t)persistent_grid(assign_delta_kernel, 256, 0));
  assign_delta_kernel<<<grid, 256, 0, st>>>(P, pnorm, n, d, C, cnorm, k, labels_prev, labels, mind, acc, state);
  PCB_CHECK_LAUNCH();
  return 0;
}

}  // namespace pcb
