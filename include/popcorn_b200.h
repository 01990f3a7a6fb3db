/*
 * popcorn_b200 — C ABI of the B200-native Lloyd hot path.
 *
 * This is the drop-in boundary below the reference's Python driver
 * `run_lloyd` (/root/reference/pkg/src/popcorn/clustering.py:291-325), which is
 * reached through the estimator plugin registry `_ALGORITHMS`
 * (estimator.py:18).  The reference binds nothing natively (it is pure
 * numpy); these are the entry points a ctypes binding of that driver calls
 * (see INTEGRATION.md).  Every function:
 *   - takes plain pointers (device pointers unless named *_host) and sizes,
 *   - takes the CUDA stream as `void*` (a cudaStream_t; NULL = legacy stream),
 *   - is asynchronous with respect to the host unless stated otherwise,
 *   - returns 0 on success, a positive cudaError_t value on a CUDA error, or a
 *     negative PCB_E* code on bad arguments (pcb_error_string() describes it).
 *
 * Per-iteration kernels read a device "state" block (int64 words: iterations
 * recorded, stop flag, converged flag, repairs of the current iteration) and
 * return immediately once the stop flag is set, so a whole max_iters loop can
 * be enqueued (or captured in a CUDA graph) with no host synchronisation —
 * the convergence test of clustering.py:322-324 runs on the device.
 *
 * Fused accumulator `acc` (f64, the buffer all-reduced across ranks):
 *   [ sums k*d | counts k | objective | changed ]   (k*d + k + 2 words)
 */
#ifndef POPCORN_B200_H
#define POPCORN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PCB_ABI_VERSION 1

#define PCB_EINVAL   (-1)   /* bad size / pointer argument            */
#define PCB_EUNSUP   (-2)   /* unsupported shape for this kernel        */
#define PCB_ENODEV   (-3)   /* no sm_100 device                          */

/* Assignment kernel variants (`variant` argument of pcb_assign_*). */
#define PCB_ASSIGN_AUTO      0  /* library picks            */
#define PCB_ASSIGN_ROWREG    1  /* FFMA, one point per thread (d <= 32)     */
#define PCB_ASSIGN_TILED     2  /* FFMA, register-tiled SIMT GEMM (any d)   */
#define PCB_ASSIGN_TC3XTF32  3  /* tcgen05 3xTF32, TMEM accumulators (f32)  */
#define PCB_ASSIGN_DELTA     4  /* delta-chunked P.C.P^T ablation (f32)     */
#define PCB_ASSIGN_SCREEN    5  /* tcgen05 1xTF32 certified screening (f32) */
#define PCB_ASSIGN_SCREEN_BF16 6 /* tcgen05 BF16 certified screening + exact candidates (f32, d <= 256) */
#define PCB_ASSIGN_SCREEN_FP8  7 /* same with E4M3 operands (kind::f8f6f4), scaled keys (f32, d <= 256) */
#define PCB_ASSIGN_DELTA_TC    8 /* delta-chunked P.C.P^T ablation on tcgen05 (3xTF32 block MMAs, f32) */

int         pcb_abi_version(void);
/* Kernels launched by this library so far in this process (launches recorded
 * into a CUDA graph count once, at capture). */
long long   pcb_launch_count(void);
const char* pcb_error_string(int code);
/* sm count / compute capability of `device`; returns PCB_ENODEV if not sm_100. */
int pcb_device_info(int device, int* sm_count, int* cc_major, int* cc_minor);

/* Input validation on the device (validation.py:45-46): *out = number of
 * non-finite entries among X[0:count]. */
int pcb_count_nonfinite_f32(const float* X, int64_t count, unsigned long long* out, void* stream);
int pcb_count_nonfinite_f64(const double* X, int64_t count, unsigned long long* out, void* stream);

/* ---- on-device init_assignments (clustering.py:91-108) --------------------
 *   labels[0:n) = Generator(PCG64(seed)).integers(0, k, size=n) as int32,
 *   then `labels[j] = j` for every empty cluster j, repeated until none is
 *   empty — bit-identical to the reference (numpy SeedSequence + PCG64 +
 *   Lemire bounded draws, see init.cu).  Synchronous (reads two ints per
 *   pass); *passes_out = number of hollow-fill passes.  Returns PCB_EUNSUP
 *   if the rejection margin is exhausted (probability ~0).
 *   pcb_pcg64_seed_state: host-only, out4 = {state hi, state lo, inc hi,
 *   inc lo} of PCG64(seed) after seeding (numpy's bit_generator.state).   */
int64_t pcb_init_scratch_bytes(int64_t n, int k);
/* The draw alone: out[0:n) = Generator(PCG64(seed)).integers(0, k, size=n)
 * (any 1 <= k < 2^31; no hollow fill).  Synchronous. */
int pcb_bounded_draws(int64_t n, int k, uint64_t seed, int32_t* out, void* scratch, int64_t scratch_bytes,
                      void* stream);
int pcb_pcg64_seed_state(uint64_t seed, uint64_t* out4_host);
int pcb_init_assignments(int64_t n, int k, uint64_t seed, int32_t* labels, void* scratch,
                         int64_t scratch_bytes, int* passes_out_host, void* stream);

/* ---- synthesized input (cli.py:102-105) ------------------------------------
 *   out[0:count) = Generator(PCG64(seed)).random(count) (row-major (n, d) when
 *   count = n*d), as f64 or rounded to f32 (.astype(f32)); bit-identical.   */
int pcb_synthesize_uniform(int64_t count, uint64_t seed, int is_f64, void* out, void* stream);

/* ---- dataset text loaders (io.py:16-77), host memory -----------------------
 *   Dense row-major n x d f32 (is_f64 = 0) or f64 into out_host (libsvm: the
 *   caller zero-fills it).  Returns 0, a positive errno if the file cannot be
 *   read, PCB_EINVAL, or PCB_EPARSE with info[4] = {kind, line number, count,
 *   text length} and the offending text (NUL-terminated) in text; kinds:
 *   1 malformed label, 2 malformed feature token, 3 feature index out of
 *   range (text = index), 4 too few libsvm lines (count = found), 5 empty CSV,
 *   6 non-numeric CSV cell (text = stripped row), 7 wrong CSV column count
 *   (count = found), 8 wrong CSV row count (count = found).
 *   nthreads <= 0: all hardware threads.                                   */
#define PCB_EPARSE   (-4)
int pcb_load_libsvm(const char* path, int64_t n, int d, int is_f64, void* out_host, int64_t* info,
                    char* text, int64_t text_len, int nthreads);
int pcb_load_csv(const char* path, int64_t n, int d, int is_f64, void* out_host, int64_t* info,
                 char* text, int64_t text_len, int nthreads);

/* ---- one-time point preparation (clustering.py:302: point_norms) ---------- */
int pcb_point_norms_f32(const float* P, int64_t n, int d, float* pnorm, void* stream);
int pcb_point_norms_f64(const double* P, int64_t n, int d, double* pnorm, void* stream);

/* Split X (rows x d, row stride d) into TF32 hi = rna_tf32(X) and lo = X - hi,
 * written with row stride `ld` (>= d, zero padded), for the 3xTF32 kernel. */
int pcb_split_tf32(const float* X, int64_t rows, int d, int ld, float* hi, float* lo, void* stream);

/* ---- assignment: distance stage + row argmin (clustering.py:310-311,
 *      dense.py:56-68) fused with the bookkeeping of _assignment_step
 *      (clustering.py:146-149): per-cluster counts and changed (the objective
 *      is summed by pcb_segment_sums_* from exact own distances).
 *   labels[i] = argmin_j D[i,j] (lowest j on ties), mind[i] = D[i,labels[i]]
 *   where D[i,j] = pnorm[i] + (cnorm[j] - 2 <p_i, c_j>).
 *   labels_prev / acc / state may be NULL (predict mode: estimator.py:131-136).
 *   C, cnorm: centroids k x d and their squared norms.
 *   For PCB_ASSIGN_TC3XTF32 the caller passes the split operands through
 *   pcb_assign_tc_f32 instead.                                              */
int pcb_assign_f32(const float* P, const float* pnorm, int64_t n, int d,
                   const float* C, const float* cnorm, int k,
                   const int32_t* labels_prev, int32_t* labels, float* mind,
                   double* acc, const long long* state, int variant, void* stream);
int pcb_assign_f64(const double* P, const double* pnorm, int64_t n, int d,
                   const double* C, const double* cnorm, int k,
                   const int32_t* labels_prev, int32_t* labels, double* mind,
                   double* acc, const long long* state, int variant, void* stream);

/* pcb_assign_f32 plus the delta update's changed-row sums: S (k x d f64, the
 * persistent per-cluster sums of pcb_delta_update_f32) gets S[new] += p,
 * S[prev] -= p for every row whose label changed, when the previous iteration
 * was a delta one, and state marks it so pcb_update_mode selects "sums
 * applied" (or discards them for a full update).  Done by the small-d
 * constant-bank kernel; other kernels leave S to pcb_delta_update_f32. */
int pcb_assign_spec_f32(const float* P, const float* pnorm, int64_t n, int d,
                        const float* C, const float* cnorm, int k,
                        const int32_t* labels_prev, int32_t* labels, float* mind,
                        double* acc, const long long* state, double* S, int variant, void* stream);

/* tcgen05 3xTF32 variant (PCB_ASSIGN_TC3XTF32): operands pre-split with
 * pcb_split_tf32 into hi/lo matrices of row stride ld (multiple of 32, >= d);
 * same outputs and bookkeeping as pcb_assign_f32.                          */
int pcb_assign_tc_f32(const float* P_hi, const float* P_lo, int ld, const float* pnorm, int64_t n,
                      int d, const float* C_hi, const float* C_lo, const float* cnorm, int k,
                      const int32_t* labels_prev, int32_t* labels, float* mind, double* acc,
                      const long long* state, void* stream);

/* delta-chunked P.C.P^T on the tensor cores (PCB_ASSIGN_DELTA_TC, the
 * tensor-core form of the attachment's scheme; see
 * assign_delta_tc.cu).  delta = 8; the augmented operands are
 *   Q   = [1, p, 0..]             n x ld          (pcb_delta_tc_prep_points, once per fit)
 *   F,G = C_j's first block column / first block row, 8 rows per centroid,
 *         (8 * pcb_delta_tc_kpad(k)) x ld    (pcb_delta_tc_prep_centroids, per iteration)
 * each split into TF32 hi + exact remainder lo; ld = pcb_delta_tc_ld(d).
 * Outputs and bookkeeping as pcb_assign_f32, with mind[i] = D[i, labels[i]]
 * (the full bilinear form, |p|^2 included).                                */
int pcb_delta_tc_ld(int d);
int pcb_delta_tc_kpad(int k);
int pcb_delta_tc_prep_points(const float* P, int64_t n, int d, int ld, float* Q_hi, float* Q_lo, void* stream);
int pcb_delta_tc_prep_centroids(const float* C, const float* cnorm, int k, int d, int ld, float* F_hi,
                                float* F_lo, float* G_hi, float* G_lo, void* stream);
int pcb_assign_delta_tc_f32(const float* Q_hi, const float* Q_lo, int ld, int64_t n, int d,
                            const float* F_hi, const float* F_lo, const float* G_hi, const float* G_lo,
                            int k, const int32_t* labels_prev, int32_t* labels, float* mind,
                            double* acc, const long long* state, void* stream);

/* Certified 1xTF32 screening variant ("tc1xtf32s", see assign_screen.cu):
 * one TF32 tensor-core pass on TF32-rounded operands (P_r = rna(P), C_r =
 * rna(C) = the finalize kernel's C_hi, row stride ld) with a rigorous per-row
 * error bound; rows whose argmin is not certified are listed in
 * amb_list/amb_count (caller zeroes amb_count) and resolved as 3xTF32 by
 * pcb_resolve_ambiguous_f32.  Labels only: counts/changed come from
 * pcb_count_labels.
 *   pcb_screen_prep_points:    P_r, anorm = |rna(p)|, danorm = |p - rna(p)|,
 *                              bstat[2] = OFF (once per fit)
 *   pcb_screen_prep_centroids: bnorm, dbnorm, bstat[0..1] (after every
 *                              centroid update)                                */
int pcb_screen_prep_points(const float* P, int64_t n, int d, int ld, float* P_r, float* anorm,
                           float* danorm, float* bstat /* 4 */, void* stream);
int pcb_screen_prep_centroids(const float* C, int k, int d, float* bnorm, float* dbnorm,
                              float* bstat, void* stream);
int pcb_assign_screen_f32(const float* P_r, int64_t n, int ld, const float* C_r, int k,
                          const float* cnorm, const float* anorm, const float* danorm,
                          const float* bstat, int32_t* labels, int* amb_list, int* amb_count,
                          const long long* state, void* stream);
/* flag_list (capacity n) / flag_count (nullable): make the resolved labels
 * exact — rows whose two best 3xTF32 keys are within the rigorous error
 * bound are re-evaluated over all k centroids (f64 sums of squares, lowest
 * index on ties) against C (f32 centroids; scratch:
 * pcb_exact_scratch_bytes()).  NULL: 3xTF32 labels.                         */
int pcb_resolve_ambiguous_f32(const float* P, int64_t n, int d, const int* amb_list,
                              const int* amb_count, int ld, float* sub_hi, float* sub_lo,
                              int32_t* sub_labels, const float* pnorm, const float* C, const float* C_hi,
                              const float* C_lo, const float* cnorm, int k, int32_t* labels,
                              int* flag_list, int* flag_count, void* scratch, int64_t scratch_bytes,
                              const long long* state, void* stream);
int64_t pcb_exact_scratch_bytes(void);   /* `scratch` of pcb_resolve_ambiguous_f32 (flag list given) */
/* Certified BF16 screening variant ("bf16s", see assign_screen_bf16.cu):
 * one BF16 tensor-core pass (kind::f16) on RN-rounded copies P_b / C_b (row
 * stride ldb = pcb_screen_bf16_ld(d) BF16 elements) with the same rigorous
 * per-row bound as the TF32 screen.  Pass 1 labels certified rows and lists
 * the others with a candidate threshold (amb_list / amb_count / amb_thr,
 * caller zeroes amb_count); pcb_resolve_screen_bf16 recomputes their keys
 * (pass 2, compact copy sub_b), collects the candidate columns (<=
 * pcb_screen_bf16_ncand() per row into cand / cand_n) and takes the exact f64
 * argmin over them.  Rows with more candidates, or all rows when amb_count >
 * bypass, are listed in ovf_list / ovf_count for pcb_resolve_ambiguous_f32.
 * Rows with exactly two keys within the bound skip pass 2: pass 1 lists them
 * in two_list as (original row, candidate, candidate) triplets (two_count,
 * caller zeroes) and the resolver evaluates both exactly.
 * labels_prev (optional) only orders the centroid tiles of each row pair
 * (the tile of the pair's previous label first); results do not depend on it.
 *   pcb_screen_prep_points_bf16:    P_b, anorm, danorm, bstat[2] = OFF (per fit)
 *   pcb_screen_prep_centroids_bf16: C_b = -2 bf16(C) (kpad rows), C_aug = |c|^2 + OFF
 *                                   as three BF16 pieces per row (the augmented K
 *                                   step: q = [p, 1], the paper's q.C.q^T form, so
 *                                   the MMA produces the ranking keys), bnorm, dbnorm,
 *                                   bstat[0..1] (per update) */
int pcb_screen_bf16_ld(int d);
int pcb_screen_bf16_ncand(void);
int pcb_screen_prep_points_bf16(const float* P, int64_t n, int d, int ldb, void* P_b, float* anorm,
                                float* danorm, float* bstat /* 16 */, void* stream);
int pcb_screen_bf16_kpad(int k);   /* rows of C_b / C_aug: k rounded up to 128 */
int pcb_screen_bf16_aug(void);     /* BF16 columns per C_aug row (16) */
int pcb_screen_prep_centroids_bf16(const float* C, const float* cnorm, int k, int d, int ldb, void* C_b,
                                   void* C_aug, float* bnorm, float* dbnorm, float* bstat, void* stream);
int pcb_assign_screen_bf16(const void* P_b, int64_t n, int ldb, const void* C_b, int k,
                           const void* C_aug, const float* anorm, const float* danorm,
                           const float* bstat, int32_t* labels, int* amb_list, int* amb_count,
                           float* amb_thr, const int32_t* orig, const int32_t* labels_prev,
                           int* two_list, int* two_count, const long long* state, void* stream);
int pcb_resolve_screen_bf16(const float* P, int64_t n, int d, const void* P_b, int ldb, const void* C_b,
                            const float* C, int k, const void* C_aug, const float* bstat,
                            const int* amb_list, const int* amb_count, const float* amb_thr,
                            int64_t bypass, void* sub_b, int* cand, int* cand_n, int32_t* labels,
                            int* ovf_list, int* ovf_count, const int32_t* orig, const int* two_list,
                            const int* two_count, const long long* state, void* stream);
/* Row layout: P_b / anorm / danorm rebuilt as the rows perm[s] of their
 * original-order copies Pb0 / an0 / dan0 (from pcb_screen_prep_points_bf16),
 * orig[s] = perm[s] (perm = point ids sorted by label, pcb_sort_by_label).
 * With orig != NULL the two calls above read P_b, anorm, danorm in that
 * layout; labels and ovf_list stay in original row ids (amb_list holds layout
 * positions).  Rows of a warp then share their nearest centroids, which lets
 * the screen skip whole 32-column chunks of its epilogue.                   */
int pcb_screen_relayout_bf16(const void* Pb0, const float* an0, const float* dan0, int64_t n, int ldb,
                             const int32_t* perm, void* P_b, float* anorm, float* danorm, int32_t* orig,
                             void* stream);
/* E4M3 screening variant ("fp8s"): the same kernels and contract as the BF16
 * one with E4M3 operand rows of ld8 = pcb_screen_fp8_ld(d) bytes (power-of-two
 * scales chosen on the device by pcb_screen_prep_points_fp8 — the points' from
 * max |p|, the centroids' from 2 max |p|, fixed for the fit; bstat of 16
 * floats; the keys are scaled by S = bstat[4] and so are amb_thr).           */
int pcb_screen_fp8_ld(int d);
int pcb_screen_prep_points_fp8(const float* P, int64_t n, int d, int ld8, void* P_q, float* anorm,
                               float* danorm, float* bstat /* 16 */, void* stream);
int pcb_screen_prep_centroids_fp8(const float* C, const float* cnorm, int k, int d, int ld8, void* C_q,
                                  void* C_aug, float* bnorm, float* dbnorm, float* bstat, void* stream);
int pcb_assign_screen_fp8(const void* P_q, int64_t n, int ld8, const void* C_q, int k, const void* C_aug,
                          const float* anorm, const float* danorm, const float* bstat, int32_t* labels,
                          int* amb_list, int* amb_count, float* amb_thr, const int32_t* orig,
                          const int32_t* labels_prev, int* two_list, int* two_count,
                          const long long* state, void* stream);
int pcb_resolve_screen_fp8(const float* P, int64_t n, int d, const void* P_q, int ld8, const void* C_q,
                           const float* C, int k, const void* C_aug, const float* bstat,
                           const int* amb_list, const int* amb_count, const float* amb_thr,
                           int64_t bypass, void* sub_q, int* cand, int* cand_n, int32_t* labels,
                           int* ovf_list, int* ovf_count, const int32_t* orig, const int* two_list,
                           const int* two_count, const long long* state, void* stream);
int pcb_count_labels(const int32_t* labels, const int32_t* labels_prev, int64_t n, int k, int d,
                     double* acc, const long long* state, void* stream);
/* The same pass fused with the delta update's changed-row sums: when the
 * previous iteration took the delta update (state[6] odd) it also applies
 * S[new] += p, S[prev] -= p for every changed row (f64 atomics) and sets
 * state[8]; pcb_update_mode then records mode 3 (delta, sums applied) or a full
 * update overwrites S.  P: n x d f32, S: k x d f64 (the S of pcb_delta_update_f32). */
int pcb_count_labels_delta_f32(const int32_t* labels, const int32_t* labels_prev, int64_t n, int k, int d,
                               double* acc, const long long* state, const float* P, double* S, void* stream);

/* ---- centroid update (clustering.py:282-288): counting sort of point ids by
 *      label, then a segmented f64 sum of point rows per cluster into acc.  */
/* counts: the counts block of acc (acc + k*d).  offsets: k+1 segment starts. */
int pcb_sort_by_label(const int32_t* labels, int64_t n, int k, const double* counts,
                      int32_t* offsets /* k+1 */, int32_t* cursor /* k */, int32_t* perm,
                      const long long* state, void* stream);
/* Adds the per-cluster row sums into acc[0 : k*d) (RED.ADD.F64) and, for
 * every sorted position s, the exact own distance own_sorted[s] =
 * sum_t (P[perm[s]][t] - C[label][t])^2 (f64) of the new labels, whose sum goes
 * to acc's objective word (clustering.py:148).  C: the centroids the labels
 * were assigned against.                                                    */
int pcb_segment_sums_f32(const float* P, int64_t n, int d, const int32_t* perm,
                         const int32_t* offsets, int k, const float* C, double* own_sorted,
                         double* acc, const long long* state, void* stream);
int pcb_segment_sums_f64(const double* P, int64_t n, int d, const int32_t* perm,
                         const int32_t* offsets, int k, const double* C, double* own_sorted,
                         double* acc, const long long* state, void* stream);

/* ---- delta centroid update (update.cu).  Per rank, S (k x d f64) holds the
 *      per-cluster sums of the rank's rows for the current labels.  After the
 *      assignment (acc holds the new local counts and changed):
 *   pcb_update_mode  -> state[6] = 1 (delta) unless force_full, more than
 *                       frac * n rows changed, a local count is 0, or a repair
 *                       marked S stale (state[7]); 0 = full update
 *   pcb_sort_by_label / pcb_segment_sums_*: no-ops in delta mode
 *   pcb_delta_update_*: delta mode: S += rows that joined, -= rows that left
 *                       (changed rows only), acc sums <- S, acc objective <-
 *                       Q - 2 sum_j <c_j, S_j> + sum_j n_j |c_j|^2 (exact
 *                       identity for sum_i |p_i - c_l(i)|^2, clustering.py:148);
 *                       full mode: S <- acc sums.  Q = pcb_sum_squares_*(P).  */
int pcb_update_mode(const double* acc, int k, int d, int64_t n, double frac, int force_full,
                    long long* state, void* stream);
int pcb_delta_update_f32(const float* P, int64_t n, int d, const int32_t* labels_prev, const int32_t* labels,
                         const float* C, int k, double* S, const double* Q, double* acc,
                         const long long* state, void* stream);
int pcb_delta_update_f64(const double* P, int64_t n, int d, const int32_t* labels_prev, const int32_t* labels,
                         const double* C, int k, double* S, const double* Q, double* acc,
                         const long long* state, void* stream);
int pcb_sum_squares_f32(const float* X, int64_t count, double* out, void* stream);
int pcb_sum_squares_f64(const double* X, int64_t count, double* out, void* stream);

/* ---- empty-cluster repair (clustering.py:111-139), single-rank, on device.
 *   For each empty cluster j ascending: the not-yet-moved point with the
 *   largest own distance (lowest index on ties) moves to j; repeated while any
 *   cluster is empty.  Reads own_sorted/perm from the update kernel, adjusts
 *   acc (sums, counts, objective, changed) and state[3] (repairs).  No-op
 *   when no cluster is empty.  One cooperative launch.  `sums` (nullable):
 *   the delta update's persistent per-cluster f64 sums, moved in step with
 *   acc; when NULL a move marks them stale (the next update runs full).   */
int64_t pcb_repair_scratch_bytes(int k);   /* device scratch the caller provides */
int pcb_repair_f32(const float* P, int64_t n, int d, const float* C, int k, const int32_t* perm,
                   const int32_t* labels_prev, int32_t* labels, double* own_sorted, double* acc,
                   long long* state, void* scratch, int64_t scratch_bytes, double* sums,
                   void* stream);
int pcb_repair_f64(const double* P, int64_t n, int d, const double* C, int k, const int32_t* perm,
                   const int32_t* labels_prev, int32_t* labels, double* own_sorted, double* acc,
                   long long* state, void* scratch, int64_t scratch_bytes, double* sums,
                   void* stream);

/* Batched multi-rank repair (one round per pass of clustering.py:126-138,
 * distributed.repair_protocol):
 *   pcb_repair_select:   this shard's E (<= 4096) unmoved points with the
 *                        largest own distance, ranked (own desc, global id
 *                        asc): out3E = E x [own, offset + id, sorted position]
 *                        (padding -inf, 9e18, -1); scratch as pcb_repair_*.
 *   pcb_repair_apply_batch_*: moves m of this rank (sorted positions pos[],
 *                        target clusters j_list[], record slots[]): labels,
 *                        own = -inf, delta records (d+4 words each, layout of
 *                        pcb_repair_apply_*) into deltas (E records, zeroed
 *                        by the caller, all-reduced SUM afterwards).
 *   pcb_repair_commit_batch: every rank applies the E records in slot order
 *                        (j_list[e] = cluster of slot e) to acc / state.
 *   pcb_flag_global_empty: after the all-reduce: if a cluster is globally
 *                        empty, saved <- acc and state[1] = 2 (repair pending:
 *                        later kernels return; the host restores acc, runs the
 *                        protocol, finalizes and clears the flag).          */
int pcb_repair_select(const double* own_sorted, const int32_t* perm, int64_t n, int64_t offset, int E,
                      double* out3E, void* scratch, int64_t scratch_bytes, void* stream);
int pcb_repair_apply_batch_f32(const float* P, int d, const float* C, const int32_t* perm,
                               const int32_t* labels_prev, int32_t* labels, double* own_sorted, const int* pos,
                               const int* j_list, const int* slots, int m, double* deltas, void* stream);
int pcb_repair_apply_batch_f64(const double* P, int d, const double* C, const int32_t* perm,
                               const int32_t* labels_prev, int32_t* labels, double* own_sorted, const int* pos,
                               const int* j_list, const int* slots, int m, double* deltas, void* stream);
int pcb_repair_commit_batch(double* acc, int k, int d, int E, const int* j_list, const double* deltas,
                            long long* state, void* stream);
int pcb_flag_global_empty(const double* acc, int k, int d, double* saved, long long* state, void* stream);

/* ---- finalize: c_j = sums_j / counts_j (empty -> 0, clustering.py:286-287),
 *      cnorm, optional TF32 hi/lo split of C (row stride ld), history
 *      recording and the convergence test (clustering.py:319-324).
 *      n_total: global point count (all ranks).                            */
int pcb_finalize_f32(const double* acc, int k, int d, int64_t n_total,
                     float* C, float* cnorm, float* c_hi, float* c_lo, int ld,
                     double* objective_hist, long long* repairs_hist,
                     long long* state, int check_convergence, double tol, void* stream);
int pcb_finalize_f64(const double* acc, int k, int d, int64_t n_total,
                     double* C, double* cnorm,
                     double* objective_hist, long long* repairs_hist,
                     long long* state, int check_convergence, double tol, void* stream);

/* Initial centroids from labels (clustering.py:298-300) without touching the
 * state: acc must hold sums+counts (sort + segment sums); writes C, cnorm. */
int pcb_centroids_from_acc_f32(const double* acc, int k, int d, float* C, float* cnorm,
                               float* c_hi, float* c_lo, int ld, void* stream);
int pcb_centroids_from_acc_f64(const double* acc, int k, int d, double* C, double* cnorm,
                               void* stream);
/* cnorm for externally supplied centroids (fixed init). */
int pcb_centroid_norms_f32(const float* C, int k, int d, float* cnorm,
                           float* c_hi, float* c_lo, int ld, void* stream);
int pcb_centroid_norms_f64(const double* C, int k, int d, double* cnorm, void* stream);

/* ==== Kernel K-means (run_popcorn, clustering.py:165-218) ====================
 * K = kernel(P P^T) is built once in HBM (row-major n x n, leading dimension
 * ldk >= n, ldk % 4 == 0 for f32 / % 2 for f64), exactly symmetric.
 * family: 0 linear, 1 polynomial, 2 gaussian, 3 sigmoid (kernels.py:18);
 * dvec = |p_i|^2 (the Gram diagonal) is required for the gaussian family.
 * *nonfinite is incremented if any K entry is not finite (require_finite).
 * pcb_kernel_gram_f32 takes the TF32 split of P (pcb_split_tf32, row stride
 * ld % 32 == 0): tcgen05 3xTF32 GEMM with the kernel in the epilogue.    */
int pcb_kernel_gram_f32(const float* P_hi, const float* P_lo, int ld, int64_t n, const float* dvec, float* K,
                        int64_t ldk, int family, double gamma, double coef, int degree, double sigma,
                        unsigned long long* nonfinite, void* stream);
int pcb_kernel_gram_f64(const double* P, int64_t n, int d, const double* dvec, double* K, int64_t ldk,
                        int family, double gamma, double coef, int degree, double sigma,
                        unsigned long long* nonfinite, void* stream);
/* Per iteration (labels_cur -> labels_new), with perm/offsets from
 * pcb_sort_by_label(labels_cur, ..., cnt, ...), cnt = counts of labels_cur (f64):
 *   segment sums  S[j, :] = sum_{m in L_j} K[m, :]  (k x lds f64, zeroed here)
 *   assign        acc = [counts k | cnsum k | objective | changed] (zeroed by
 *                 the caller); D[i,j] = K[i,i] - 2 S[j,i]/|L_j| + c_j,
 *                 c_j = (1/|L_j|) sum_{i in L_j} S[l_i,i]/|L_{l_i}|; argmin
 *                 -> labels_new, own distance, int counts (icounts)
 *   repair        empty clusters filled by the farthest points (one block)
 *   finalize      counts/objective/changed of labels_new, history at
 *                 state[0], convergence; cnt <- counts of labels_new.     */
int pcb_kk_segment_sums_f32(const float* K, int64_t ldk, int64_t n, int64_t ncols, const int32_t* perm,
                            const int32_t* offsets, int k, double* S, int64_t lds, const long long* state,
                            void* stream);
int pcb_kk_segment_sums_f64(const double* K, int64_t ldk, int64_t n, int64_t ncols, const int32_t* perm,
                            const int32_t* offsets, int k, double* S, int64_t lds, const long long* state,
                            void* stream);
int pcb_kk_assign_f32(const float* K, int64_t ldk, const double* S, int64_t lds, int64_t n, int k,
                      const double* cnt, double* acc, const int32_t* labels_cur, int32_t* labels_new, double* own,
                      int* icounts, long long* state, void* stream);
int pcb_kk_assign_f64(const double* K, int64_t ldk, const double* S, int64_t lds, int64_t n, int k,
                      const double* cnt, double* acc, const int32_t* labels_cur, int32_t* labels_new, double* own,
                      int* icounts, long long* state, void* stream);
int64_t pcb_kk_repair_scratch_bytes(int64_t n, int k);
int pcb_kk_repair_f32(const float* K, int64_t ldk, const double* S, int64_t lds, int64_t n, int k,
                      const double* cnt, const double* acc, int32_t* labels, double* own, int* icounts,
                      long long* state, void* scratch, int64_t scratch_bytes, void* stream);
int pcb_kk_repair_f64(const double* K, int64_t ldk, const double* S, int64_t lds, int64_t n, int k,
                      const double* cnt, const double* acc, int32_t* labels, double* own, int* icounts,
                      long long* state, void* scratch, int64_t scratch_bytes, void* stream);
/* Rectangular kernel matrix K (na x nb, leading dimension ldk) = kernel(A B^T)
 * (kernels.py:143-166 kernel_matrix_between: no pinned gaussian diagonal);
 * dva/dvb = squared row norms (gaussian only).  f32 takes TF32 splits.     */
int pcb_kernel_cross_f32(const float* A_hi, const float* A_lo, int64_t na, const float* B_hi, const float* B_lo,
                         int64_t nb, int ld, const float* dva, const float* dvb, float* K, int64_t ldk, int family,
                         double gamma, double coef, int degree, double sigma, unsigned long long* nonfinite,
                         void* stream);
int pcb_kernel_cross_f64(const double* A, int64_t na, const double* B, int64_t nb, int d, const double* dva,
                         const double* dvb, double* K, int64_t ldk, int family, double gamma, double coef, int degree,
                         double sigma, unsigned long long* nonfinite, void* stream);
/* predict (estimator.py:131-147): out[i] = argmin_j self_i - 2 S[j,i]/|L_j| + cself_j
 * with S from pcb_kk_segment_sums over the cross matrix (training rows by
 * label), xn = |x_i|^2 and cself_j = sum_{l,m in L_j} K(l,m) / |L_j|^2.     */
int pcb_kk_predict_f32(const double* S, int64_t lds, int64_t m, int k, const double* cnt, const double* cself,
                       const float* xn, int family, double gamma, double coef, int degree, double sigma,
                       int32_t* out, void* stream);
int pcb_kk_predict_f64(const double* S, int64_t lds, int64_t m, int k, const double* cnt, const double* cself,
                       const double* xn, int family, double gamma, double coef, int degree, double sigma,
                       int32_t* out, void* stream);
int pcb_kk_finalize(const int32_t* labels, const int32_t* labels_prev, const double* own, int64_t n, int k,
                    double* acc, double* cnt, double* obj_hist, long long* rep_hist, long long* state,
                    int check_convergence, double tol, void* stream);

/* ==== Tensor-core accumulation probe (test infrastructure) ==================
 * One chain of tcgen05.mma steps, M = N = 128, 32 bytes of K per step, F32
 * accumulator in TMEM: D = init + sum_s A_s B_s^T (init may be NULL).  A, B:
 * 128 rows of nsteps*32 bytes each (K contiguous); kinds[s] (device ints):
 * 0 E4M3 (kind::f8f6f4, K=32), 1 BF16 (kind::f16, K=16), 2 TF32 (kind::tf32,
 * K=8).  D: 128 x 128 f32, row-major.  Measures the rounding model the
 * screening certificates assume (tests/test_gpu_mma_probe.py).             */
int pcb_mma_probe(const void* A, const void* B, const int* kinds, int nsteps, const float* init, float* D,
                  void* stream);
/* Same chain with every step E4M3 into an F16 accumulator (the F16-key
 * screen): init (f32, rounded to f16, may be NULL) is written and D read back
 * through tcgen05.st/ld .unpack/.pack::16b; raw (may be NULL) receives the
 * 128 x 128 unpacked 32-bit TMEM cells (layout check).                       */
int pcb_mma_probe_f16acc(const void* A, const void* B, const int* kinds, int nsteps, const float* init, float* D,
                         uint32_t* raw, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* POPCORN_B200_H */
