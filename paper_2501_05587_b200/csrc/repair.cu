// Empty-cluster repair on the device (clustering.py:111-139, called from
// _assignment_step clustering.py:146).
//
// Semantics reproduced exactly: while some cluster is empty, for each cluster
// that was empty at the start of the pass, in ascending order, the point with
// the largest own distance D[i, label_i] among points not moved yet (ties ->
// lowest index) is moved to that cluster.  Own distances of unmoved points
// never change (their labels do not), so own_sorted[] written by the update
// kernel (in label-sorted order, perm[s] = point id) is the reference's `own`
// vector; a moved point gets own = -inf.
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

// Exact own distance (same evaluation as the update kernel): sum (p - c)^2 in f64.
template <typename T>
__device__ double pair_distance(const T* P, const T* C, int d, int64_t i, int j) {
  double q = 0.0;
  for (int t = 0; t < d; ++t) {
    const double e = (double)P[i * d + t] - (double)C[(int64_t)j * d + t];
    q = fma(e, e, q);
  }
  return q;
}


// Donors of one pass are the top-E unmoved points in (own distance desc,
// point id asc) order: every argmax of the reference's loop excludes the points
// taken before it and no other own distance changes, so the e-th donor is the
// e-th point of that order.  Selection: a 12-digit radix select over the
// 96-bit key (ordered own bits, ~point id) finds the B-th largest key (B =
// empties handled in this batch, <= RP_BATCH), a scan collects the B keys at or
// above it, block 0 ranks them, and all blocks apply the B moves at once.
// ~0.3 ms per batch at n = 10M instead of one grid-wide argmax (and two grid
// barriers) per empty cluster.
constexpr int RP_BATCH = 4096;

struct RepairScratch {
  unsigned long long hist[3][256];
  int sel_count;
  int pad;
  unsigned long long sel_k1[RP_BATCH];
  unsigned int sel_k2[RP_BATCH];
  int sel_q[RP_BATCH];
  int move_q[RP_BATCH];  // sorted position of the e-th donor
  int elist[1];          // [0] = #empty, then the empty clusters ascending (k entries)
};

__device__ __forceinline__ unsigned long long own_key(double v) {
  return (unsigned long long)ordered_bits(v);  // total order, -inf (taken) smallest
}

// Select mode (sel_out != nullptr; multi-rank repair, see pcb_repair_select):
// no accumulator, no moves — one batch of B = sel_E selections whose ranked
// keys (own distance, offset + point id, sorted position) go to sel_out.
template <typename T>
__global__ void __launch_bounds__(256)
repair_kernel(const T* __restrict__ P, int64_t n, int d, const T* __restrict__ C, int k,
              const int32_t* __restrict__ perm, const int32_t* __restrict__ labels_prev,
              int32_t* __restrict__ labels, double* __restrict__ own, double* __restrict__ acc,
              long long* __restrict__ state, RepairScratch* __restrict__ sc, double* __restrict__ S,
              int sel_E = 0, double* __restrict__ sel_out = nullptr, long long offset = 0) {
  const bool select = sel_out != nullptr;
  if (!select && stopped(state)) return;
  cg::grid_group grid = cg::this_grid();
  const AccLayout L{k, d};
  __shared__ int s_any;
  __shared__ unsigned int s_hist[256];
  __shared__ unsigned long long s_glob[256];
  __shared__ int s_wsum[8];
  if (threadIdx.x == 0) s_any = select ? 1 : 0;
  __syncthreads();
  if (!select)
    for (int j = threadIdx.x; j < k; j += blockDim.x)
      if (acc[L.counts() + j] == 0.0) s_any = 1;
  __syncthreads();
  if (!s_any) return;  // identical decision in every block: no barrier reached

  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = (int64_t)blockIdx.x * per, hi = min(n, lo + per);
  int hbuf = 0;  // triple-buffered global histograms (the next pass's zeroed during this one)
  if (blockIdx.x == 0)
    for (int i = threadIdx.x; i < 3 * 256; i += blockDim.x) (&sc->hist[0][0])[i] = 0ull;
  while (true) {
    grid.sync();  // counts of the previous pass are final
    if (select) {
      if (blockIdx.x == 0 && threadIdx.x == 0) sc->elist[0] = min(sel_E, RP_BATCH);
    } else if (blockIdx.x == 0) {  // ascending list of the empty clusters (block-wide ballot scan)
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      int base = 0;
      for (int j0 = 0; j0 < k; j0 += blockDim.x) {
        const int j = j0 + threadIdx.x;
        const bool e = j < k && acc[L.counts() + j] == 0.0;
        const unsigned int bal = __ballot_sync(0xffffffffu, e);
        if (lane == 0) s_wsum[warp] = __popc(bal);
        __syncthreads();
        int off = base;
        for (int w = 0; w < warp; ++w) off += s_wsum[w];
        if (e) sc->elist[1 + off + __popc(bal & ((1u << lane) - 1u))] = j;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) base += s_wsum[w];
        __syncthreads();
      }
      if (threadIdx.x == 0) sc->elist[0] = base;
    }
    grid.sync();
    const int ne = ((volatile int*)sc->elist)[0];
    if (ne == 0) break;
    for (int e0 = 0; e0 < ne; e0 += RP_BATCH) {
      const int B = min(RP_BATCH, ne - e0);
      // ---- radix select of the B-th largest key over the unmoved points
      unsigned long long p1 = 0ull, m1 = 0ull;  // prefix / mask on the own bits
      unsigned int p2 = 0u, m2 = 0u;            // prefix / mask on ~point id
      int rem = B;
      for (int pass = 0; pass < 12; ++pass) {
        const int nb = (hbuf + 1) % 3;
        if (blockIdx.x == 0)  // buffer of the next pass: last read two passes ago (before the last barrier)
          for (int i = threadIdx.x; i < 256; i += blockDim.x) sc->hist[nb][i] = 0ull;
        for (int i = threadIdx.x; i < 256; i += blockDim.x) s_hist[i] = 0u;
        __syncthreads();
        // 4 loads in flight per thread (the pass is a latency-bound stream over own[])
        for (int64_t b0 = lo; b0 < hi; b0 += 4 * (int64_t)blockDim.x) {  // block-uniform trip count
          const int64_t q0 = b0 + threadIdx.x;
          unsigned long long kk[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int64_t q = q0 + (int64_t)u * blockDim.x;
            kk[u] = q < hi ? own_key(own[q]) : 0ull;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int64_t q = q0 + (int64_t)u * blockDim.x;
            const unsigned long long k1 = kk[u];
            bool hit = q < hi && (k1 & m1) == p1;
            unsigned int dig = 0u;
            if (hit) {
              if (pass < 8) {
                dig = (unsigned int)(k1 >> (8 * (7 - pass))) & 255u;
              } else {
                const unsigned int k2 = ~(unsigned int)perm[q];
                hit = (k2 & m2) == p2;
                dig = (k2 >> (8 * (11 - pass))) & 255u;
              }
            }
            // warp-aggregated: the leading digits are shared by most rows
            const unsigned int peers = __match_any_sync(0xffffffffu, hit ? dig : 0xffffffffu);
            if (hit && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&s_hist[dig], (unsigned)__popc(peers));
          }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < 256; i += blockDim.x)
          if (s_hist[i]) atomicAdd(&sc->hist[hbuf][i], (unsigned long long)s_hist[i]);
        grid.sync();
        // every block scans the global histogram from the top (same result);
        // one parallel load into shared memory, then a serial scan there
        for (int i = threadIdx.x; i < 256; i += blockDim.x)
          s_glob[i] = ((volatile unsigned long long*)sc->hist[hbuf])[i];
        __syncthreads();
        if (threadIdx.x == 0) {
          unsigned long long cum = 0ull;
          int bsel = 0;
          for (int bb = 255; bb >= 0; --bb) {
            const unsigned long long c = s_glob[bb];
            if (cum + c >= (unsigned long long)rem) { bsel = bb; break; }
            cum += c;
          }
          s_hist[0] = (unsigned int)bsel;
          s_hist[1] = (unsigned int)(rem - (int)cum);
          s_hist[2] = (unsigned int)(s_glob[bsel] == (unsigned long long)(rem - (int)cum));  // whole bucket taken
        }
        __syncthreads();
        const unsigned int bsel = s_hist[0];
        rem = (int)s_hist[1];
        const bool whole = s_hist[2] != 0u;
        __syncthreads();
        if (pass < 8) {
          p1 |= (unsigned long long)bsel << (8 * (7 - pass));
          m1 |= 255ull << (8 * (7 - pass));
        } else {
          p2 |= bsel << (8 * (11 - pass));
          m2 |= 255u << (8 * (11 - pass));
        }
        hbuf = nb;
        if (whole) break;  // every key of the selected bucket is among the B: prefix suffices
      }
      // the B largest keys are those whose (masked) prefix is >= (p1, p2) (ids
      // are unique; a shorter prefix only when its whole bucket is selected)
      if (blockIdx.x == 0 && threadIdx.x == 0) sc->sel_count = 0;
      grid.sync();
      for (int64_t q = lo + threadIdx.x; q < hi; q += blockDim.x) {
        const unsigned long long k1 = own_key(own[q]);
        if ((k1 & m1) < p1) continue;
        const unsigned int k2 = ~(unsigned int)perm[q];
        if ((k1 & m1) == p1 && (k2 & m2) < p2) continue;
        const int at = atomicAdd(&sc->sel_count, 1);
        if (at < RP_BATCH) { sc->sel_k1[at] = k1; sc->sel_k2[at] = k2; sc->sel_q[at] = (int)q; }
      }
      grid.sync();
      // block 0 ranks them: rank e -> donor of the (e0 + e)-th empty cluster
      if (blockIdx.x == 0) {
        const int cnt = min(((volatile int*)&sc->sel_count)[0], B);
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
          const unsigned long long a1 = sc->sel_k1[i];
          const unsigned int a2 = sc->sel_k2[i];
          int r = 0;
          for (int j = 0; j < cnt; ++j) {
            const unsigned long long b1 = sc->sel_k1[j];
            r += (b1 > a1) || (b1 == a1 && sc->sel_k2[j] > a2);
          }
          sc->move_q[r] = sc->sel_q[i];
        }
      }
      grid.sync();
      if (select) {  // ranked keys out, nothing moved
        const int cnt = min(((volatile int*)&sc->sel_count)[0], B);
        if (blockIdx.x == 0)
          for (int e = threadIdx.x; e < B; e += blockDim.x) {
            const bool ok = e < cnt;
            const int q = ok ? sc->move_q[e] : -1;
            sel_out[3 * e + 0] = ok ? own[q] : -INFINITY;
            sel_out[3 * e + 1] = ok ? (double)(offset + perm[q]) : 9.0e18;
            sel_out[3 * e + 2] = (double)q;
          }
        return;
      }
      // apply the B moves, one warp per move
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      const int cntm = min(((volatile int*)&sc->sel_count)[0], B);
      for (int e = blockIdx.x * (int)(blockDim.x >> 5) + warp; e < cntm; e += gridDim.x * (int)(blockDim.x >> 5)) {
        const int64_t q = sc->move_q[e];
        const int j = sc->elist[1 + e0 + e];
        const int64_t donor = perm[q];
        const int old = labels[donor];
        for (int t = lane; t < d; t += 32) {
          const double p = (double)P[donor * d + t];
          atomicAdd(&acc[(int64_t)old * d + t], -p);
          atomicAdd(&acc[(int64_t)j * d + t], p);
          if (S != nullptr) {  // keep the delta update's per-cluster sums in step
            atomicAdd(&S[(int64_t)old * d + t], -p);
            atomicAdd(&S[(int64_t)j * d + t], p);
          }
        }
        if (lane == 0) {
          const double dnew = pair_distance(P, C, d, donor, j);
          atomicAdd(&acc[L.objective()], dnew - own[q]);
          if (labels_prev != nullptr) {
            const int prev = labels_prev[donor];
            atomicAdd(&acc[L.changed()], (double)((j != prev) - (old != prev)));
          }
          atomicAdd(&acc[L.counts() + old], -1.0);
          atomicAdd(&acc[L.counts() + j], 1.0);
          labels[donor] = j;
          own[q] = -INFINITY;
          atomicAdd((unsigned long long*)&state[kMoved], 1ull);
          if (S == nullptr) state[kSumsStale] = 1;  // the delta update's per-cluster sums miss this move
        }
      }
      grid.sync();  // own / labels of the moves visible to the next selection
    }
  }
}

// Cooperative grid: up to 4 blocks per SM (the selection passes stream own[]).
static int repair_grid(int per_sm) { return sm_count() * std::min(per_sm, 4); }

static size_t repair_scratch(int k) { return sizeof(RepairScratch) + sizeof(int) * (size_t)(k + 1); }

template <typename T>
static int repair(const T* P, int64_t n, int d, const T* C, int k, const int32_t* perm,
                  const int32_t* lp, int32_t* lab, double* own, double* acc, long long* state,
                  void* scratch, int64_t scratch_bytes, double* S, cudaStream_t st) {
  if (n < 1 || d < 1 || k < 1 || !P || !C || !perm || !lab || !own || !acc || !state || !scratch)
    return PCB_EINVAL;
  if (n > INT32_MAX) return PCB_EUNSUP;
  if (scratch_bytes < (int64_t)repair_scratch(k)) return PCB_EINVAL;
  auto kern = repair_kernel<T>;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
  if (e != cudaSuccess) return (int)e;
  if (per_sm < 1) return PCB_EUNSUP;
  const int grid = repair_grid(per_sm);
  RepairScratch* sc = (RepairScratch*)scratch;
  int sel_E = 0;
  double* sel_out = nullptr;
  long long offset = 0;
  void* args[] = {(void*)&P,   (void*)&n,   (void*)&d,   (void*)&C,     (void*)&k,
                  (void*)&perm, (void*)&lp, (void*)&lab, (void*)&own, (void*)&acc,
                  (void*)&state, (void*)&sc, (void*)&S, (void*)&sel_E, (void*)&sel_out, (void*)&offset};
  pcb::count_launch();
  e = cudaLaunchCooperativeKernel((void*)kern, dim3(grid), dim3(256), args, 0, st);
  return (int)e;
}

// Select mode launch: the E (<= RP_BATCH) unmoved points of this shard with
// the largest own distance, ranked (own desc, global id asc), as
// [own, offset + id, sorted position] triplets; padding (-inf, 9e18, -1).
static int repair_select(const double* own, const int32_t* perm, int64_t n, int64_t offset, int E, double* out,
                         void* scratch, int64_t scratch_bytes, cudaStream_t st) {
  if (n < 1 || E < 1 || E > RP_BATCH || !own || !perm || !out || !scratch) return PCB_EINVAL;
  if (n > INT32_MAX) return PCB_EUNSUP;
  if (scratch_bytes < (int64_t)repair_scratch(1)) return PCB_EINVAL;
  auto kern = repair_kernel<float>;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
  if (e != cudaSuccess) return (int)e;
  if (per_sm < 1) return PCB_EUNSUP;
  const int grid = repair_grid(per_sm);
  RepairScratch* sc = (RepairScratch*)scratch;
  const float* P = nullptr;
  const float* C = nullptr;
  int d = 1, k = 1;
  const int32_t* lp = nullptr;
  int32_t* lab = nullptr;
  double* ownp = const_cast<double*>(own);
  double* acc = nullptr;
  long long* state = nullptr;
  double* S = nullptr;
  long long off = offset;
  void* args[] = {(void*)&P,    (void*)&n,   (void*)&d,     (void*)&C,  (void*)&k,  (void*)&perm,
                  (void*)&lp,   (void*)&lab, (void*)&ownp,  (void*)&acc, (void*)&state, (void*)&sc,
                  (void*)&S,    (void*)&E,   (void*)&out,   (void*)&off};
  pcb::count_launch();
  e = cudaLaunchCooperativeKernel((void*)kern, dim3(grid), dim3(256), args, 0, st);
  return (int)e;
}

}  // namespace pcb

extern "C" int64_t pcb_repair_scratch_bytes(int k) { return (int64_t)pcb::repair_scratch(k); }

extern "C" int pcb_repair_select(const double* own_sorted, const int32_t* perm, int64_t n, int64_t offset, int E,
                                 double* out3E, void* scratch, int64_t scratch_bytes, void* stream) {
  return pcb::repair_select(own_sorted, perm, n, offset, E, out3E, scratch, scratch_bytes, (cudaStream_t)stream);
}

extern "C" int pcb_repair_f32(const float* P, int64_t n, int d, const float* C, int k,
                              const int32_t* perm, const int32_t* labels_prev, int32_t* labels,
                              double* own_sorted, double* acc, long long* state, void* scratch,
                              int64_t scratch_bytes, double* sums, void* stream) {
  return pcb::repair<float>(P, n, d, C, k, perm, labels_prev, labels, own_sorted, acc, state, scratch,
                            scratch_bytes, sums, (cudaStream_t)stream);
}

extern "C" int pcb_repair_f64(const double* P, int64_t n, int d, const double* C, int k,
                              const int32_t* perm, const int32_t* labels_prev, int32_t* labels,
                              double* own_sorted, double* acc, long long* state, void* scratch,
                              int64_t scratch_bytes, double* sums, void* stream) {
  return pcb::repair<double>(P, n, d, C, k, perm, labels_prev, labels, own_sorted, acc, state, scratch,
                            scratch_bytes, sums, (cudaStream_t)stream);
}

// ---------------------------------------------------------------------------
// Multi-rank repair building blocks (host-orchestrated, rare path; see
// distributed.repair_protocol).  Delta record of one move (f64, d+4 words):
//   [ p_donor (d) | old label | d_objective | d_changed | valid ]
// ---------------------------------------------------------------------------
namespace pcb {

// Batched multi-rank moves: move m (one warp each) takes the donor at sorted
// position pos[m] to cluster jl[m] and writes its delta record to slot sl[m]
// of `deltas` (E records of d+4 words; the caller zeroes them, so after the
// all-reduce every slot holds its owner's record).
template <typename T>
__global__ void repair_apply_batch_kernel(const T* __restrict__ P, int d, const T* __restrict__ C,
                                          const int32_t* __restrict__ perm, const int32_t* __restrict__ labels_prev,
                                          int32_t* __restrict__ labels, double* __restrict__ own,
                                          const int* __restrict__ pos, const int* __restrict__ jl,
                                          const int* __restrict__ sl, int m, double* __restrict__ deltas) {
  const int lane = threadIdx.x & 31;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int e = w0; e < m; e += nw) {
    const int64_t q = pos[e];
    const int j = jl[e];
    const int64_t donor = perm[q];
    double* rec = deltas + (int64_t)sl[e] * (d + 4);
    double part = 0.0;
    for (int t = lane; t < d; t += 32) {
      const double p = (double)P[donor * d + t];
      rec[t] = p;
      const double df = p - (double)C[(int64_t)j * d + t];
      part = fma(df, df, part);
    }
    part = warp_sum(part);
    if (lane == 0) {
      const int old = labels[donor];
      rec[d] = (double)old;
      rec[d + 1] = part - own[q];
      rec[d + 2] = labels_prev ? (double)((j != labels_prev[donor]) - (old != labels_prev[donor])) : 0.0;
      rec[d + 3] = 1.0;
      labels[donor] = j;
      own[q] = -INFINITY;
    }
  }
}

// Every rank applies the E all-reduced records in slot order (one block, so
// every rank rounds the same way and the accumulators stay identical).
__global__ void repair_commit_batch_kernel(double* __restrict__ acc, int k, int d, int E, const int* __restrict__ jl,
                                           const double* __restrict__ deltas, long long* __restrict__ state) {
  const AccLayout L{k, d};
  for (int e = 0; e < E; ++e) {
    const double* rec = deltas + (int64_t)e * (d + 4);
    if (rec[d + 3] != 1.0) continue;
    const int old = (int)rec[d], j = jl[e];
    for (int t = threadIdx.x; t < d; t += blockDim.x) {
      acc[(int64_t)old * d + t] -= rec[t];
      acc[(int64_t)j * d + t] += rec[t];
    }
    if (threadIdx.x == 0) {
      acc[L.counts() + old] -= 1.0;
      acc[L.counts() + j] += 1.0;
      acc[L.objective()] += rec[d + 1];
      acc[L.changed()] += rec[d + 2];
      state[kMoved] += 1;
      state[kSumsStale] = 1;
    }
    __syncthreads();
  }
}

// Multi-rank: after the all-reduce, a globally empty cluster makes this
// iteration wait for the host's repair protocol — the accumulator is saved
// and state[kStop] = 2 (every later kernel of the iteration and of the
// iterations already enqueued returns at once; the host restores the
// accumulator, repairs, finalizes and resumes; engine.ShardSequence).
__global__ void __launch_bounds__(1024)
flag_global_empty_kernel(const double* __restrict__ acc, int k, int d, double* __restrict__ saved,
                         long long* __restrict__ state) {
  if (stopped(state)) return;
  const AccLayout L{k, d};
  __shared__ int any;
  if (threadIdx.x == 0) any = 0;
  __syncthreads();
  for (int j = threadIdx.x; j < k; j += blockDim.x)
    if (acc[L.counts() + j] == 0.0) any = 1;
  __syncthreads();
  if (!any) return;
  for (int64_t i = threadIdx.x; i < L.size(); i += blockDim.x) saved[i] = acc[i];
  __syncthreads();
  if (threadIdx.x == 0) state[kStop] = 2;
}

}  // namespace pcb

extern "C" int pcb_repair_apply_batch_f32(const float* P, int d, const float* C, const int32_t* perm,
                                          const int32_t* labels_prev, int32_t* labels, double* own_sorted,
                                          const int* pos, const int* j_list, const int* slots, int m, double* deltas,
                                          void* stream) {
  if (d < 1 || m < 0 || !P || !C || !perm || !labels || !own_sorted || !deltas || (m && (!pos || !j_list || !slots)))
    return PCB_EINVAL;
  if (m == 0) return 0;
  pcb::repair_apply_batch_kernel<float><<<std::min(1024, (m + 7) / 8), 256, 0, (cudaStream_t)stream>>>(
      P, d, C, perm, labels_prev, labels, own_sorted, pos, j_list, slots, m, deltas);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_repair_apply_batch_f64(const double* P, int d, const double* C, const int32_t* perm,
                                          const int32_t* labels_prev, int32_t* labels, double* own_sorted,
                                          const int* pos, const int* j_list, const int* slots, int m, double* deltas,
                                          void* stream) {
  if (d < 1 || m < 0 || !P || !C || !perm || !labels || !own_sorted || !deltas || (m && (!pos || !j_list || !slots)))
    return PCB_EINVAL;
  if (m == 0) return 0;
  pcb::repair_apply_batch_kernel<double><<<std::min(1024, (m + 7) / 8), 256, 0, (cudaStream_t)stream>>>(
      P, d, C, perm, labels_prev, labels, own_sorted, pos, j_list, slots, m, deltas);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_repair_commit_batch(double* acc, int k, int d, int E, const int* j_list, const double* deltas,
                                       long long* state, void* stream) {
  if (k < 1 || d < 1 || E < 1 || !acc || !j_list || !deltas || !state) return PCB_EINVAL;
  pcb::repair_commit_batch_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(acc, k, d, E, j_list, deltas, state);
  PCB_CHECK_LAUNCH();
  return 0;
}

extern "C" int pcb_flag_global_empty(const double* acc, int k, int d, double* saved, long long* state,
                                     void* stream) {
  if (k < 1 || d < 1 || !acc || !saved || !state) return PCB_EINVAL;
  pcb::flag_global_empty_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(acc, k, d, saved, state);
  PCB_CHECK_LAUNCH();
  return 0;
}
