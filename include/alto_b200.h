/*
 * alto_b200.h -- C ABI of the B200-native ALTO hot path.
 *
 * The reference (pkg/src/alto, Python + numba) has no C ABI: its hot loops are
 * numba functions with a caller-owned-buffer convention (pkg/src/alto/_jit.py).
 * Each entry point below replaces one of those loops or one of the numpy
 * vectorised stages that feed them; the reference symbol is cited per entry.
 *
 * Conventions
 *   - Every pointer is a DEVICE pointer unless its name starts with host_.
 *   - `stream` is a cudaStream_t passed as void*; all work is stream-ordered
 *     and asynchronous unless stated otherwise.
 *   - Every call returns an alto_status (0 = OK). alto_last_error() gives a
 *     thread-local message for the last failure. The Python shim maps
 *     ALTO_ERR_VALUE -> ValueError, ALTO_ERR_INDEX -> IndexError,
 *     ALTO_ERR_UNSUPPORTED -> UnsupportedShapeError, ALTO_ERR_NUMERICAL ->
 *     NumericalError, ALTO_ERR_CUDA -> RuntimeError (reference error contract:
 *     pkg/src/alto/validation.py:8-64).
 *   - Positions (keys) are uint64[M] for layouts of <= 64 bits and
 *     uint64[M][2] = {low word, high word} otherwise, exactly the reference
 *     storage (pkg/src/alto/tensor.py:133-138).
 *   - Factor matrices are fp64, row-major, row stride `ld` doubles
 *     (ld >= rank; the shim pads to a multiple of 4 for 32-byte rows).
 */
#ifndef ALTO_B200_H
#define ALTO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ALTO_MAX_MODES 16
#define ALTO_MAX_SPANS 192

typedef enum {
  ALTO_OK = 0,
  ALTO_ERR_VALUE = 1,
  ALTO_ERR_INDEX = 2,
  ALTO_ERR_UNSUPPORTED = 3,
  ALTO_ERR_NUMERICAL = 4,
  ALTO_ERR_CUDA = 5
} alto_status;

/* Bit layout: per-mode spans already split at 64-bit word edges
 * (reference: AltoLayout + _split_word_spans, pkg/src/alto/encoding.py:90-114,
 * :213-225). Span s of mode n (span_off[n] <= s < span_off[n+1]) copies
 * span_len[s] bits from coordinate bit span_src[s] to bit span_bit[s] of key
 * word span_word[s]. */
typedef struct alto_layout_t {
  int32_t nmodes;
  int32_t word_bits; /* 64 or 128 */
  int32_t total_bits;
  int32_t nspans;
  int64_t dims[ALTO_MAX_MODES];
  int32_t span_off[ALTO_MAX_MODES + 1];
  uint8_t span_src[ALTO_MAX_SPANS];
  uint8_t span_bit[ALTO_MAX_SPANS];
  uint8_t span_len[ALTO_MAX_SPANS];
  uint8_t span_word[ALTO_MAX_SPANS];
} alto_layout_t;

/* Factor matrices of one model (the reference stacks them per call with
 * np.vstack, pkg/src/alto/kernels.py:145-148; here they stay separate). */
typedef struct alto_factors_t {
  int32_t nmodes;
  int32_t rank;
  const double *ptr[ALTO_MAX_MODES];
  int64_t ld[ALTO_MAX_MODES];
} alto_factors_t;

/* MTTKRP / Phi fast-path algorithms over the ALTO-ordered stream. */
typedef enum {
  ALTO_ALGO_ATOMIC = 0,     /* direct fp64 global reductions (red.global.add.f64) */
  ALTO_ALGO_PRIVATIZED = 1  /* per-segment shared-memory output privatisation */
} alto_algo;

int alto_abi_version(void);
const char *alto_last_error(void);
int alto_device_sm_count(int32_t *host_sms);

/* ---- encoder --------------------------------------------------------- */

/* Bit-gather linearisation of coords[M][N] (int64) into keys.
 * Replaces encode_coords (pkg/src/alto/encoding.py:228-247). Out-of-range
 * coordinates: *host_bad_row receives the first offending row (or -1), the
 * call returns ALTO_ERR_INDEX (synchronises the stream). */
int alto_encode(const alto_layout_t *host_layout, const int64_t *coords,
                int64_t M, void *keys, int64_t *host_bad_row, void *stream);

/* Bit-scatter back to coords[M][N] (int64).
 * Replaces decode_coords (pkg/src/alto/encoding.py:250-262). */
int alto_decode(const alto_layout_t *host_layout, const void *keys, int64_t M,
                int64_t *coords, void *stream);

/* Scratch size for alto_sort_pairs / alto_canonicalize. */
int alto_sort_scratch_bytes(int64_t M, int32_t word_bits, size_t *host_bytes);

/* Ascending sort of (key, value) pairs by key, in place, stable; only the
 * low total_bits bits are significant.
 * Replaces argsort(kind="stable") / lexsort((lo, hi)) in AltoTensor.from_coo
 * (pkg/src/alto/tensor.py:201-205, :210). */
int alto_sort_pairs(const alto_layout_t *host_layout, void *keys, double *vals,
                    int64_t M, void *scratch, size_t scratch_bytes, void *stream);

/* Canonicalise keys produced under a lexicographic layout: stable sort,
 * sum duplicates in input order, drop exact zeros; compacts keys/vals in
 * place and writes the surviving count to *host_M_out (synchronises).
 * Replaces CooTensor._canonicalize (pkg/src/alto/tensor.py:116-124). */
int alto_canonicalize(const alto_layout_t *host_lex_layout, void *keys,
                      double *vals, int64_t M, void *scratch,
                      size_t scratch_bytes, int64_t *host_M_out, void *stream);

/* Range and finiteness validation of a COO input (synchronises).
 * host_flags[0] = first out-of-range row or -1; host_flags[1] = first
 * non-finite value row or -1. (pkg/src/alto/tensor.py:72-78) */
int alto_validate_coo(const int64_t *coords, const double *vals, int64_t M,
                      int32_t N, const int64_t *host_dims, int64_t *host_flags,
                      void *stream);

/* Gather-rate probe (B200 addition, measurement only): random 128-byte row
 * gathers from a table of table_rows rows (dview3's access pattern, all
 * SMs), reps timed launches; writes rows per second. The ceiling the
 * decoded-view kernels are measured against (bench.py roofline.gather). */
int alto_gather_probe(int32_t table_rows, int32_t reps, double *host_rows_per_s);

/* Deterministic mode of the fast decoded-view kernels (MTTKRP and Phi over
 * unblocked decoded views, the memoised sweep): row runs cut by a segment
 * edge are parked per segment and folded in a fixed order instead of fp64
 * reductions, so repeated calls give bitwise identical results (the
 * reference's own order is the exact=True path). Process-wide; the edge
 * slots are allocated on first use (not inside a graph capture). */
int alto_set_deterministic(int32_t on);
int alto_get_deterministic(int32_t *host_on);

/* ---- partitioning ---------------------------------------------------- */

/* Balanced line segments: bounds[L+1] (balanced_bounds) and per-segment,
 * per-mode tight intervals lo/hi[L][N] of the decoded coordinates.
 * Replaces balanced_bounds + make_segments' reduceat
 * (pkg/src/alto/partition.py:69-75, :91-95). */
int alto_partition(const alto_layout_t *host_layout, const void *keys,
                   int64_t M, int32_t L, int64_t *bounds, int64_t *lo,
                   int64_t *hi, void *stream);

/* Per-row first/last segment id for one mode (rows in >= 2 segments are
 * boundary rows). row_min/row_max must be int32[dims[mode]]; they are
 * initialised by the call. Replaces _rows_spanning_segments
 * (pkg/src/alto/partition.py:117-120, :126-134). */
int alto_row_segment_span(const alto_layout_t *host_layout, const void *keys,
                          int64_t M, int32_t mode, const int64_t *bounds,
                          int32_t L, int32_t *row_min, int32_t *row_max,
                          void *stream);

/* counts[i] = number of the M ascending keys strictly below queries[i]
 * (same word format as keys; 128-bit keys compare the high word first).
 * The splitter search of the distributed construction (SURVEY.md 8(e):
 * shard boundaries equal to the single-GPU balanced_bounds) runs on it. */
int alto_count_less(int32_t word_bits, const void *keys, int64_t M,
                    const void *queries, int32_t nq, int64_t *counts,
                    void *stream);

/* Mode-ordered view: stable sort of the ALTO-ordered stream by the mode-n
 * coordinate. Writes perm[M] (int64, index into the ALTO order), and the
 * permuted keys and values. Replaces make_mode_ordered_view's argsort
 * (pkg/src/alto/partition.py:185-188). */
int alto_mode_view(const alto_layout_t *host_layout, const void *keys,
                   const double *vals, int64_t M, int32_t mode, int64_t *perm,
                   void *view_keys, double *view_vals, void *scratch,
                   size_t scratch_bytes, void *stream);
int alto_mode_view_scratch_bytes(int64_t M, size_t *host_bytes);

/* ---- MTTKRP ------------------------------------------------------------ */

/* Fast MTTKRP over the ALTO-ordered stream: out[I_mode][ldo] += ...
 * (out must be zeroed by the caller). algo must be ALTO_ALGO_ATOMIC (the
 * segment tables are ignored); the privatised algorithm is
 * alto_mttkrp_segment below. Replaces mttkrp_sequential / mttkrp_recursive hot loops
 * (pkg/src/alto/kernels.py:160-210, pkg/src/alto/_jit.py:16-30, :53-64). */
int alto_mttkrp_stream(const alto_layout_t *host_layout, const void *keys,
                       const double *vals, int64_t M,
                       const alto_factors_t *host_factors, int32_t mode,
                       double *out, int64_t ldo, int32_t algo,
                       const int64_t *bounds, const int64_t *lo, int32_t L,
                       void *stream);

/* ALTO line-segment MTTKRP with shared-memory output privatisation, the
 * paper's conflict resolution (reference recursive
 * strategy pkg/src/alto/kernels.py:169-210, _jit.py:16-30, :53-64).
 * One CTA per segment l of alto_partition's tables (bounds[L+1], lo[L][N]):
 * the segment's keys are streamed in ALTO order and decoded in registers;
 * privatize != 0: the output interval [lo_l, lo_l + acc_rows) x R lives in
 * shared memory (acc_rows >= every segment's interval width) and is added to
 * `out` once per segment with fp64 reductions; privatize == 0: row runs of
 * the tile-local row order are reduced into `out` directly. `out` must be
 * zeroed. 3..5 modes, dims < 2^32. alto_segment_smem_bytes reports the shared
 * memory a privatised launch needs (ALTO_ERR_UNSUPPORTED above the device's
 * per-block limit). */
int alto_segment_smem_bytes(int32_t word_bits, int32_t nmodes, int32_t rank,
                            int64_t acc_rows, size_t *host_bytes);
int alto_mttkrp_segment(const alto_layout_t *host_layout, const void *keys,
                        const double *vals, int64_t M,
                        const alto_factors_t *host_factors, int32_t mode,
                        double *out, int64_t ldo, const int64_t *bounds,
                        const int64_t *lo, int32_t L, int64_t acc_rows,
                        int32_t privatize, void *stream);

/* Exact-order MTTKRP, bit-identical to the reference's recursive strategy
 * with the same L (L = 1 is the sequential strategy): per-segment private
 * buffers accumulated in ALTO order, then a pull reduction in ascending
 * segment order. temps must hold sum_l (hi_l - lo_l + 1) * rank doubles and
 * be zeroed; seg_offs[L] (int64) are the per-segment offsets into temps.
 * (pkg/src/alto/_jit.py:16-30, :53-64; pkg/src/alto/kernels.py:187-210) */
int alto_mttkrp_exact(const alto_layout_t *host_layout, const void *keys,
                      const double *vals, int64_t M,
                      const alto_factors_t *host_factors, int32_t mode,
                      double *out, int64_t ldo, const int64_t *bounds,
                      const int64_t *lo, const int64_t *hi,
                      const int64_t *seg_offs, int32_t L, double *temps,
                      void *stream);

/* Output-oriented MTTKRP over a mode-ordered view (rows contiguous) split
 * into L balanced segments: each segment's row runs are accumulated in
 * registers in view order and written once; runs cut by a segment edge are
 * parked in per-segment edge slots (scratch, alto_run_scratch_bytes(L)) and
 * folded in ascending segment order. For the reference's L the result is
 * bit-identical to mttkrp_output_oriented (its boundary rows / side buffers,
 * pkg/src/alto/kernels.py:213-252, pkg/src/alto/_jit.py:33-50) when
 * exact != 0 (no FMA contraction); exact == 0 allows FMA.
 * `out` must be zeroed (rows without nonzeros stay zero). */
int alto_mttkrp_oriented(const alto_layout_t *host_layout,
                         const void *view_keys, const double *view_vals,
                         int64_t M, const alto_factors_t *host_factors,
                         int32_t mode, double *out, int64_t ldo, int64_t L,
                         int32_t exact, void *scratch, size_t scratch_bytes,
                         void *stream);

/* Edge scratch for L segments, and the segment count the fast path uses
 * for an M-nonzero stream. */
int alto_run_scratch_bytes(int64_t L, size_t *host_bytes);
int alto_default_segments(int64_t M, int64_t *host_nseg);

/* ---- CP-APR ------------------------------------------------------------ */

/* Khatri-Rao rows Pi[M][ldp] = prod_{m != mode, ascending} A_m[i_m, :]
 * (pkg/src/alto/cpd/apr.py:101-111). */
int alto_pi(const alto_layout_t *host_layout, const void *keys, int64_t M,
            const alto_factors_t *host_factors, int32_t mode, double *pi,
            int64_t ldp, void *stream);

/* Phi (model-update ratio) over the ALTO stream, fast path:
 *   out[i] += v / max(scaled[i] . krp, eps) * krp
 * krp from pi (PRE, ldp > 0) or recomputed from the factors (OTF, pi NULL).
 * (pkg/src/alto/cpd/apr.py:114-180, pkg/src/alto/_jit.py:67-102) */
int alto_phi_stream(const alto_layout_t *host_layout, const void *keys,
                    const double *vals, int64_t M,
                    const alto_factors_t *host_factors, int32_t mode,
                    const double *scaled, int64_t lds, const double *pi,
                    int64_t ldp, double eps, double *out, int64_t ldo,
                    int32_t algo, const int64_t *bounds, const int64_t *lo,
                    int32_t L, void *stream);

/* Exact-order Phi, bit-identical to the reference's sequential/recursive
 * strategies with the same L (same temps convention as alto_mttkrp_exact). */
int alto_phi_exact(const alto_layout_t *host_layout, const void *keys,
                   const double *vals, int64_t M,
                   const alto_factors_t *host_factors, int32_t mode,
                   const double *scaled, int64_t lds, const double *pi,
                   int64_t ldp, double eps, double *out, int64_t ldo,
                   const int64_t *bounds, const int64_t *lo, const int64_t *hi,
                   const int64_t *seg_offs, int32_t L, double *temps,
                   void *stream);

/* Output-oriented Phi over a mode-ordered view (pi, if given, must already
 * be permuted into view order; pkg/src/alto/cpd/apr.py:171-179,
 * pkg/src/alto/_jit.py:105-137). The scaled row is loaded once per row run.
 * exact != 0: sequential rank dot and no FMA (bit-identical to the
 * reference for the same L). rank <= 32. */
int alto_phi_oriented(const alto_layout_t *host_layout, const void *view_keys,
                      const double *view_vals, int64_t M,
                      const alto_factors_t *host_factors, int32_t mode,
                      const double *scaled, int64_t lds, const double *pi,
                      int64_t ldp, double eps, double *out, int64_t ldo,
                      int64_t L, int32_t exact, void *scratch,
                      size_t scratch_bytes, void *stream);

/* Fused inner-iteration epilogue of cp_apr_mu
 * (pkg/src/alto/cpd/apr.py:183-185, :300-310):
 *   kkt = max |min(b, 1 - phi)|   over rows x rank
 *   if apply: b *= phi (stores into b) and flags non-finite results.
 * host_out[0] = kkt, host_out[1] = 1.0 if a non-finite product was produced.
 * `apply` < 0 means: apply iff kkt >= tau (device-side decision). Synchronises. */
int alto_apr_update(double *b, int64_t ldb, const double *phi, int64_t ldphi,
                    int64_t rows, int32_t rank, double tau, int32_t apply,
                    double *host_out, void *stream);

/* Poisson log-likelihood data term sum_x v_x * log(mhat_x),
 * mhat_x = sum_r lambda_r prod_n A_n[i_n, r] (the rank sum in ascending r).
 * Writes one partial per block into partials (>= alto_loglik_partials())
 * and the fixed-order total into *host_sum (synchronises).
 * (pkg/src/alto/cpd/apr.py:200-207, pkg/src/alto/cpd/model.py:66-72) */
int alto_loglik(const alto_layout_t *host_layout, const void *keys,
                const double *vals, int64_t M,
                const alto_factors_t *host_factors, const double *lambda,
                double *partials, double *host_sum, void *stream);
int alto_loglik_partials(int64_t M, int32_t *host_count);

/* Device-driven CP-APR inner loop (B200 addition). The reference decides
 * after every Phi whether to stop (pkg/src/alto/cpd/apr.py:290-310: Phi,
 * kkt = max|min(B, 1 - Phi)|, break if kkt < tau, else B *= Phi). Here the
 * decision stays on the device: reset a state block, enqueue max_inner
 * iterations of { alto_zero_if(Phi); alto_phi_dview(..., skip = state);
 * alto_apr_inner_step(iter) } without host round trips (every kernel is a
 * no-op once the loop is done), then read the outcome once. */
int alto_apr_inner_state_bytes(int32_t max_inner, size_t *host_bytes);
int alto_apr_inner_reset(void *state, void *stream);
/* Byte offset of the per-iteration KKT values (double[max_inner]) in the
 * state block; the state starts with int32 {done, 1 + first non-finite
 * iteration, iterations used}. Lets a caller copy results asynchronously. */
int alto_apr_inner_kkt_offset(size_t *host_offset);
int alto_zero_if(double *out, int64_t ld, int64_t rows, const void *state,
                 void *stream);
/* dst[0:n] = src[0:n] unless the loop is done (multi-GPU device loop: the
 * reduced Phi of the last executed iteration is kept for the next outer
 * iteration's shift while the collective keeps running on skipped ones). */
int alto_copy_if(const double *src, double *dst, int64_t n, const void *state,
                 void *stream);
int alto_apr_inner_step(double *b, int64_t ldb, const double *phi,
                        int64_t ldphi, int64_t rows, int32_t rank, double tau,
                        int32_t iter, void *state, void *stream);
/* Synchronises: iterations used, 1 + first non-finite iteration (0: none),
 * and the KKT value of the last iteration performed. */
int alto_apr_inner_result(const void *state, int32_t *host_used,
                          int32_t *host_nonfinite_iter, double *host_kkt,
                          void *stream);

/* CP-ALS factor update for one mode on the device (B200 addition; replaces
 * the host steps of pkg/src/alto/cpd/als.py:115-124 and
 * pkg/src/alto/cpd/linalg.py:11-52): V = Hadamard product of the other
 * modes' Grams (grams: nmodes x rank x rank, device), upper Cholesky of V,
 * a = mt V^-1 by the two triangular solves (written to `a`, row stride
 * lda), weights = column norms of a, a /= norms (0 -> 1), grams[mode] =
 * a^T a. flags[0] |= 1 on non-finite input, flags[1] |= 1 when V is not
 * positive definite (the caller falls back to the pseudo-inverse on the
 * host). rank <= 32. Stream-ordered, no host sync (graph-capturable). */
int alto_als_update_scratch_bytes(int64_t rows, int32_t rank,
                                  size_t *host_bytes);
int alto_als_update(const double *mt, int64_t ldm, int64_t rows, int32_t rank,
                    double *grams, int32_t nmodes, int32_t mode, double *a,
                    int64_t lda, double *weights, void *scratch,
                    size_t scratch_bytes, int32_t *flags, void *stream);
/* The same update split in two so the Cholesky of mode n's normal matrix
 * (which needs only the Gram matrices, final after mode n-1's update) can
 * run on another stream while mode n's MTTKRP runs: alto_als_chol writes
 * the factor into the scratch block, alto_als_update_solve(do_chol = 0)
 * uses it (do_chol = 1: same as alto_als_update). */
int alto_als_chol(const double *grams, int32_t nmodes, int32_t mode, int32_t rank,
                  void *scratch, size_t scratch_bytes, int32_t *flags, void *stream);
/* The update for a row block when the rows of mode n are owned by several
 * ranks (multi-GPU: reduce-scatter of the MTTKRP partials to row owners):
 * alto_als_solve_gram solves the block's rows and writes the block's raw
 * Gram a^T a (rank x rank, before normalisation) to gram_raw; the caller
 * sums gram_raw over ranks (the column norms are sqrt(diag)), then
 * alto_als_normalize writes weights, grams[mode] = G / (s s^T) and scales
 * the block's rows by 1/s; the blocks are then all-gathered. The solve is
 * row-separable (mt V^-1), so this equals the single-GPU update up to the
 * summation order of the Gram. */
int alto_als_solve_gram(const double *mt, int64_t ldm, int64_t rows, int32_t rank,
                        const double *grams, int32_t nmodes, int32_t mode, double *a,
                        int64_t lda, void *scratch, size_t scratch_bytes, int32_t *flags,
                        int32_t do_chol, double *gram_raw, void *stream);
int alto_als_normalize(const double *gram_raw, int32_t rank, double *grams,
                       int32_t nmodes, int32_t mode, double *a, int64_t lda,
                       int64_t rows, double *weights, void *scratch,
                       size_t scratch_bytes, void *stream);
int alto_als_update_solve(const double *mt, int64_t ldm, int64_t rows, int32_t rank,
                          double *grams, int32_t nmodes, int32_t mode, double *a,
                          int64_t lda, double *weights, void *scratch,
                          size_t scratch_bytes, int32_t *flags, int32_t do_chol,
                          void *stream);

/* Finiteness of factor matrices (B200 addition; the device side of
 * check_factors, pkg/src/alto/validation.py:30-57, for factors uploaded from
 * host memory): flags[n] (device, nmodes int32) = 1 when mode n's
 * host_rows[n] x rank matrix holds a non-finite entry, else 0; mode `skip`
 * (-1: none) is not scanned. Stream-ordered: the caller reads the flags back
 * with the result of the kernel that consumed the factors. */
int alto_factors_nonfinite(const alto_factors_t *host_factors,
                           const int64_t *host_rows, int32_t skip,
                           int32_t *flags, void *stream);
/* Upload host factors (row stride host_ld doubles) into the device copies
 * of dev_factors for every mode but `skip`, then alto_factors_nonfinite
 * (flags may be NULL: no scan). */
int alto_upload_factors(const alto_factors_t *dev_factors,
                        const double *const *host_ptrs, const int64_t *host_rows,
                        int32_t host_ld, int32_t skip, int32_t *flags, void *stream);
/* cudaMemsetAsync(ptr, 0, bytes) on the stream. */
int alto_memset_async(void *ptr, size_t bytes, void *stream);

/* FROSTT text ingestion (host, multi-threaded; the canonicalisation that
 * follows runs on the GPU through alto_canonicalize). Restates parse_frostt
 * (pkg/src/alto/tensor.py:245-296): one-based indices then a value per line,
 * '#' comments and blank lines skipped, mode count from the first data line.
 * Errors return ALTO_ERR_VALUE with the reference's message in
 * alto_last_error() and the 1-based line in *host_err_line (-1: none).
 * `threads` <= 0 uses every hardware thread. */
int alto_frostt_scan(const char *host_text, int64_t len, int32_t threads,
                     int64_t *host_entries, int32_t *host_ndim,
                     int64_t *host_err_line);
int alto_frostt_parse(const char *host_text, int64_t len, int32_t threads,
                      int32_t ndim, int64_t entries, int64_t *host_coords,
                      double *host_values, int64_t *host_err_line);

/* ------------------------------------------------------------------------
 * Decoded mode views (B200 additions; same results as the oriented path,
 * a different in-HBM layout). A mode view (alto_mode_view) is decoded once
 * into rows[M] (u32 target-mode coordinate) and crd (u32, N-1 planes of
 * stride round_up(M, 8), the other modes ascending) so the hot kernels read
 * 4 + 4(N-1) + 8 bytes per nonzero instead of the key + vals and skip the
 * per-nonzero bit extraction. Dims must be < 2^32. Replaces the per-call
 * mode-ordered view walk of pkg/src/alto/kernels.py:213-252 (MTTKRP) and
 * pkg/src/alto/cpd/apr.py:98-121 (Phi) for the fast (non-exact) path.
 * Any view order works (the kernels only need rows grouped); the shim
 * decodes the fiber view (alto_fiber_view) for N >= 3, whose sub-order by
 * the shortest other mode makes consecutive nonzeros share a factor row. */
int alto_decode_view(const alto_layout_t *host_layout, const void *view_keys,
                     int64_t M, int32_t mode, uint32_t *rows, uint32_t *crd,
                     void *stream);
/* MTTKRP / Phi over a decoded view: fixed 512-nonzero segments, row runs in
 * registers, segment-edge rows with red.global.add.f64 (fast, FMA allowed).
 * rows_recur != 0 (blocked views, where a row has one run per block): every
 * run is reduced with red.global.add.f64.
 * fiber_plane is ignored (kept for ABI stability; the fiber-factored
 * variant measured slower and was removed).
 * `out` must be zeroed. Phi's pi (ldp) may be NULL (computed on the fly).
 * `skip` (nullable) is an alto_apr_inner state: the launch is a no-op once
 * that loop is done. */
/* Memoised CP-ALS sweep (3-mode tensors; modes m0 then m1 in sweep order,
 * k the third mode). Pieces = runs of equal (row, m1 coordinate) inside the
 * 512-nonzero segments of m0's decoded fiber view sorted by (row, m1).
 * alto_memo_pieces_count: per-segment counts and their exclusive scan
 * pbase[nseg + 1] (P = pbase[nseg]). alto_memo_pieces_build: the consumer
 * order (pieces sorted by (m1 coordinate, row)): prow/pcrd per position and
 * pid[position] = piece (keys/ids: P u64 each; scratch per
 * alto_memo_sort_scratch_bytes). alto_mttkrp_memo0: MTTKRP of m0 that also
 * stores T[piece] = sum v * A_k[k] per piece, pieces in view order
 * (ldT = a multiple of 4 >= rank). alto_mttkrp_memo1: MTTKRP of m1 = sum
 * over positions A_m0[pcrd] o T[pid] into rows prow (valid while A_k is
 * unchanged since memo0). `out` zeroed. */
int alto_memo_pieces_count(const uint32_t *rows, const uint32_t *jcrd, int64_t M,
                           uint32_t *counts, uint32_t *pbase, void *stream);
int alto_memo_sort_scratch_bytes(int64_t P, size_t *host_bytes);
int alto_memo_pieces_build(const uint32_t *rows, const uint32_t *jcrd, int64_t M,
                           const uint32_t *pbase, int64_t P, int64_t nrows_m0,
                           int64_t nrows_m1, uint64_t *keys, uint64_t *ids,
                           void *scratch, size_t scratch_bytes, uint32_t *prow,
                           uint32_t *pcrd, uint32_t *pid, void *stream);
int alto_mttkrp_memo0(const alto_layout_t *host_layout, const uint32_t *rows,
                      const uint32_t *crd, const double *vals, int64_t M,
                      const alto_factors_t *host_factors, int32_t mode,
                      int32_t next_mode, const uint32_t *pbase, double *T,
                      int64_t ldT, double *out, int64_t ldo, void *stream);
/* pid == NULL: the pieces are walked in T order (position == piece). */
/* Interleaved streams (csrc/memo_sums.cu): elements per field of the
 * zero-padded interleaved layout of an M-nonzero stream for `rank`. */
int alto_il_length(int64_t M, int32_t rank, int64_t *host_len);
/* Fused branch-free producer: T[p] as alto_memo_sums_fast (T == NULL: not
 * stored) and out[i] += A_j[j_p] o T[p] for this mode's MTTKRP (`out`
 * zeroed). Stream by alto_memo_fused_stream: rows, j | piece-start << 31, k,
 * vals, interleaved (alto_il_length elements each). */
int alto_memo_fused_stream(const uint32_t *rows, const uint32_t *jcrd, const uint32_t *kcrd,
                           const double *vals, int64_t M, int32_t rank, uint32_t *il_rows,
                           uint32_t *il_jf, uint32_t *il_k, double *il_vals, void *stream);
int alto_memo_fused(const uint32_t *il_rows, const uint32_t *il_jf, const uint32_t *il_k,
                    const double *il_vals, int64_t M, const double *Aj, int64_t ldj,
                    const double *Ak, int64_t ldk, int32_t rank, const uint32_t *pbase,
                    const uint32_t *il_pos, double *T, int64_t ldT, double *out, int64_t ldo,
                    void *stream);
/* Fused fiber-factored MTTKRP of a 3-5 mode tensor: alto_fused_stream_n packs a
 * decoded fiber view of the mode (rows, nplanes = N - 1 coordinate planes of
 * stride crd_ld in ascending mode order, the fiber mode's plane `jplane`,
 * values; view order: sorted by (row, fiber coordinate)) into the
 * interleaved stream (rows, j | piece start << 31, the N - 2 other planes at
 * stride alto_il_length(M, rank), values); alto_mttkrp_fused then gathers the
 * fiber mode's row (Aj) once per (row, fiber) piece and the nk = N - 2 other
 * rows (Ak[t], host array of device pointers, ascending modes) per nonzero.
 * `out` zeroed; rank <= 32, dims < 2^31. */
int alto_fused_stream_n(const uint32_t *rows, const uint32_t *crd, int64_t crd_ld, int32_t nplanes,
                        int32_t jplane, const double *vals, int64_t M, int32_t rank,
                        uint32_t *il_rows, uint32_t *il_jf, uint32_t *il_k, double *il_vals,
                        void *stream);
/* The same interleaved stream built straight from the ALTO tensor in one call:
 * the stable sort by (mode coordinate, fiber-mode coordinate) of
 * alto_fiber_view (reference pkg/src/alto/partition.py:185-188) followed by
 * one pass that gathers keys and values through the sort's permutation,
 * decodes the other N - 2 coordinates in registers and writes the stream --
 * no permuted key copy and no decoded view in between (bit-identical to
 * alto_fiber_view + alto_decode_view + alto_fused_stream_n). `perm`: int64[M]
 * work array; scratch as alto_mode_view_scratch_bytes(M). view_rows /
 * view_fiber (both or neither, u32[M]): also receive the view's row and
 * fiber-mode coordinates in view order (the memoised plan's piece index,
 * alto_memo_pieces_count / _build / alto_memo_fused_pos, is built from them). */
int alto_fused_stream_build(const alto_layout_t *host_layout, const void *keys, const double *vals,
                            int64_t M, int32_t mode, int32_t fiber_mode, int32_t rank, int64_t *perm,
                            uint32_t *il_rows, uint32_t *il_jf, uint32_t *il_k, double *il_vals,
                            uint32_t *view_rows, uint32_t *view_fiber, void *scratch,
                            size_t scratch_bytes, void *stream);
int alto_mttkrp_fused(const uint32_t *il_rows, const uint32_t *il_jf, const uint32_t *il_k,
                      const double *il_vals, int64_t M, int32_t nk, const double *Aj, int64_t ldj,
                      const double *const *Ak, const int64_t *ldk, int32_t rank, double *out,
                      int64_t ldo, void *stream);
/* Consumer-ordered piece sums. alto_memo_consumer_layout lays the consumer's
 * pieces (prow = output row, pcrd = gathered row, pid = T-order piece id, in
 * consumer order) out in the consumer's interleaved layout
 * (alto_memo_consumer_length(P, rank) slots) and returns every piece's slot;
 * alto_memo_fused_pos marks the producer stream's piece starts with their
 * slots (il_pos, alto_il_length(M, rank) elements), so alto_memo_fused with
 * il_pos stores T[p] at its slot (T: consumer_length rows); alto_memo_consume
 * then streams T: out[j] = sum_pieces A[i] o T[p] (`out` zeroed). */
int alto_memo_consumer_length(int64_t P, int32_t rank, int64_t *host_len);
int alto_memo_consumer_layout(const uint32_t *prow, const uint32_t *pcrd, const uint32_t *pid,
                              int64_t P, int32_t rank, uint32_t *il_prow, uint32_t *il_pcrd,
                              uint32_t *slot_of_piece, void *stream);
int alto_memo_fused_pos(const uint32_t *rows, const uint32_t *jcrd, int64_t M,
                        const uint32_t *pbase, const uint32_t *slot_of_piece, int32_t rank,
                        uint32_t *il_pos, void *stream);
int alto_memo_consume(const uint32_t *il_prow, const uint32_t *il_pcrd, const double *T,
                      int64_t ldT, int64_t P, const double *A, int64_t lda, int32_t rank,
                      double *out, int64_t ldo, void *stream);
/* Call memo of the public mttkrp() (memo.CallMemo; B200 addition, the
 * reference recomputes every call, pkg/src/alto/kernels.py:284-303): a T
 * stored by a producing call is valid for any later call whose A_k equals,
 * bitwise, the A_k it was produced with (T depends on the tensor and A_k
 * only). alto_memo_key_check sets *flag (device int32) to valid && A == key
 * over the first `rank` columns of `rows` rows; the _if variants of the
 * producer / consumer run iff (*flag != 0) == run_if, so the choice between
 * them stays on the device; alto_memo_key_save copies A into key iff
 * (*pred != 0) == save_if (pred NULL: always). */
int alto_memo_key_check(const double *A, int64_t lda, const double *key, int64_t ldk,
                        int64_t rows, int32_t rank, int32_t valid, int32_t *flag,
                        void *stream);
int alto_memo_key_save(const double *A, int64_t lda, double *key, int64_t ldk,
                       int64_t rows, int32_t rank, const int32_t *pred, int32_t save_if,
                       void *stream);
int alto_memo_fused_if(const uint32_t *il_rows, const uint32_t *il_jf, const uint32_t *il_k,
                       const double *il_vals, int64_t M, const double *Aj, int64_t ldj,
                       const double *Ak, int64_t ldk, int32_t rank, const uint32_t *pbase,
                       const uint32_t *il_pos, double *T, int64_t ldT, double *out,
                       int64_t ldo, const int32_t *pred, int32_t run_if, void *stream);
int alto_memo_consume_if(const uint32_t *il_prow, const uint32_t *il_pcrd, const double *T,
                         int64_t ldT, int64_t P, const double *A, int64_t lda, int32_t rank,
                         double *out, int64_t ldo, const int32_t *pred, int32_t run_if,
                         void *stream);
int alto_mttkrp_memo1(const uint32_t *prow, const uint32_t *pcrd, const uint32_t *pid,
                      const double *T, int64_t ldT, int64_t P, const double *A, int64_t lda,
                      int32_t rank, double *out, int64_t ldo, void *stream);
int alto_mttkrp_dview(const alto_layout_t *host_layout, const uint32_t *rows,
                      const uint32_t *crd, const double *vals, int64_t M,
                      const alto_factors_t *host_factors, int32_t mode,
                      int32_t rows_recur, int32_t fiber_plane, double *out,
                      int64_t ldo, void *stream);
int alto_phi_dview(const alto_layout_t *host_layout, const uint32_t *rows,
                   const uint32_t *crd, const double *vals, int64_t M,
                   const alto_factors_t *host_factors, int32_t mode,
                   int32_t rows_recur, int32_t fiber_plane,
                   const double *scaled, int64_t lds,
                   const double *pi,
                   int64_t ldp, double eps, double *out, int64_t ldo,
                   const void *skip, double *pi_il_out, void *stream);
/* Streamed-Pi Phi (CP-APR inner iterations 2..max_inner of a mode; replaces
 * the gathers of phi_kernel's OTF path, pkg/src/alto/cpd/apr.py:114-180, by a
 * stream of the Khatri-Rao rows, which are fixed inside a mode's inner loop).
 * Layout: the decoded view's 512-nonzero segments in blocks of 32 (lane =
 * segment % 32); slot (block, j, lane); Pi column c of a slot at
 * (block*512 + j)*rank*32 + c*32 + lane. alto_phi_dview(pi_il_out != NULL)
 * writes Pi in this layout while it computes Phi (rank <= 16, pi == NULL).
 * alto_pstream_build copies the view's rows/values into slot order (once per
 * mode). alto_phi_pstream: `out` zeroed; `skip` as alto_phi_dview. */
int alto_pstream_sizes(int64_t M, int32_t rank, int64_t *host_slots,
                       int64_t *host_pi_doubles);
int alto_pstream_build(const uint32_t *rows, const double *vals, int64_t M,
                       uint32_t *il_rows, double *il_vals, void *stream);
/* Poisson log-likelihood data term sum_x v_x log(<scaled[row_x], Pi[x]>)
 * from streamed Khatri-Rao rows (scaled = lambda o A_mode; Pi of `mode`
 * stored with the current factors of the other modes). partials: device
 * double[alto_loglik_pstream_partials()]; the total lands in partials[0]
 * (fixed-order sums: deterministic for a given device). */
int alto_loglik_pstream_partials(int32_t *host_count);
int alto_loglik_pstream(const uint32_t *il_rows, const double *il_vals,
                        const double *pi_il, int64_t M, int32_t rank,
                        const double *scaled, int64_t lds, double *partials,
                        int32_t partials_count, void *stream);
/* Compact slot layout for count data (every value an integer in [0, 255],
 * the mode < 65536 rows): u16 rows and u8 values per slot (83 instead of 92
 * bytes per nonzero at R = 10); alto_phi_pstream2 / alto_loglik_pstream2 take
 * either layout (compact = 1: il_rows are uint16_t, il_vals uint8_t). */
int alto_pstream_build_compact(const uint32_t *rows, const double *vals, int64_t M,
                               uint16_t *il_rows, uint8_t *il_vals, void *stream);
int alto_phi_pstream2(const void *il_rows, const void *il_vals, int32_t compact,
                      const double *pi_il, int64_t M, int32_t rank, int32_t rows_recur,
                      const double *scaled, int64_t lds, double eps, double *out, int64_t ldo,
                      const void *skip, void *stream);
int alto_loglik_pstream2(const void *il_rows, const void *il_vals, int32_t compact,
                         const double *pi_il, int64_t M, int32_t rank, const double *scaled,
                         int64_t lds, double *partials, int32_t partials_count, void *stream);
int alto_phi_pstream(const uint32_t *il_rows, const double *il_vals,
                     const double *pi_il, int64_t M, int32_t rank,
                     int32_t rows_recur, const double *scaled, int64_t lds,
                     double eps, double *out, int64_t ldo, const void *skip,
                     void *stream);
/* Fiber view: the stream stably sorted by (mode, fiber_mode) coordinates
 * (scratch as alto_mode_view_scratch_bytes); decoded by alto_decode_view. */
int alto_fiber_view(const alto_layout_t *host_layout, const void *keys,
                    const double *vals, int64_t M, int32_t mode,
                    int32_t fiber_mode, int64_t *perm, void *view_keys,
                    double *view_vals, void *scratch, size_t scratch_bytes,
                    void *stream);
/* Khatri-Rao rows of a decoded view in view order (the PRE rows of the
 * decoded-view Phi): pi[x] = prod_{m != mode} A_m[i_m], ascending mode order
 * (precompute_krp_rows, pkg/src/alto/cpd/apr.py:101-111). */
int alto_pi_dview(const alto_layout_t *host_layout, const uint32_t *rows,
                  const uint32_t *crd, int64_t M,
                  const alto_factors_t *host_factors, int32_t mode, double *pi,
                  int64_t ldp, void *stream);

/* Poisson log-likelihood data term over a decoded view of `mode`:
 * sum_x v_x log(<scaled[i_mode], prod_{m != mode} A_m[i_m]>) with scaled =
 * lambda o A_mode (rows x lds). Writes per-block partials and, at index
 * count - 1 (alto_loglik_dview_partials), the fixed-order total; no host
 * sync. Replaces the values_at pass of pkg/src/alto/cpd/apr.py:200-207. */
int alto_loglik_dview_partials(int64_t M, int32_t rank, int32_t *host_count);
int alto_loglik_dview(const alto_layout_t *host_layout, const uint32_t *rows,
                      const uint32_t *crd, const double *vals, int64_t M,
                      const alto_factors_t *host_factors, int32_t mode,
                      const double *scaled, int64_t lds, double *partials,
                      void *stream);

/* Blocked fiber view: sorted by (coordinate of block_mode >> block_shift,
 * mode coordinate, fiber_mode coordinate), stable. Blocks of the largest
 * other mode keep that factor's rows L1-resident while a block is walked;
 * a row then has one run per block (kernels take rows_recur = 1). */
int alto_blocked_view(const alto_layout_t *host_layout, const void *keys,
                      const double *vals, int64_t M, int32_t mode,
                      int32_t fiber_mode, int32_t block_mode,
                      int32_t block_shift, int64_t *perm, void *view_keys,
                      double *view_vals, void *scratch, size_t scratch_bytes,
                      void *stream);

/* ------------------------------------------------------------------------
 * NCCL-aware entries (SURVEY.md 8(b) "alto_mttkrp_sharded(..., ncclComm_t)",
 * 8(e)). The reference is one process (pkg/src/alto/kernels.py:130-142 fans
 * a call out over threads); these are the multi-GPU form of the same calls.
 * NCCL is resolved at run time (the process's libnccl.so.2, e.g. the one
 * torch.distributed loaded); without it every entry returns
 * ALTO_ERR_UNSUPPORTED. `comm` is an ncclComm_t passed as void*; the
 * collectives are enqueued on `stream` (capturable in CUDA graphs) and fail
 * with ALTO_ERR_CUDA (RuntimeError), e.g. after a peer aborted.
 *
 * alto_nccl_unique_id: rank 0 makes the id (host_len >= 128 bytes) and ships
 * it to the other ranks out of band (torch.distributed broadcast in the
 * shim); alto_nccl_comm_init is collective over the `world` ranks (call with
 * the rank's device current). alto_nccl_check reports an asynchronous
 * communicator error; destroy with abort != 0 tears a broken communicator
 * down without waiting for peers. */
int alto_nccl_version(int32_t *host_version);
int alto_nccl_unique_id(uint8_t *host_id, int64_t host_len);
int alto_nccl_comm_init(const uint8_t *host_id, int64_t host_len, int32_t world,
                        int32_t rank, void **host_comm);
int alto_nccl_comm_destroy(void *comm, int32_t abort);
int alto_nccl_comm_info(void *comm, int32_t *host_world, int32_t *host_rank);
int alto_nccl_check(void *comm);
/* In-place sum over the ranks of count doubles. */
int alto_nccl_allreduce_f64(double *buf, int64_t count, void *comm, void *stream);
/* recv (recvcount doubles) = rank r's block of the sum of every rank's send
 * (world * recvcount doubles); in place when recv = send + r * recvcount. */
int alto_nccl_reduce_scatter_f64(const double *send, double *recv,
                                 int64_t recvcount, void *comm, void *stream);
/* recv (world * sendcount doubles) = every rank's send block, rank order. */
int alto_nccl_allgather_f64(const double *send, double *recv, int64_t sendcount,
                            void *comm, void *stream);
/* Sharded MTTKRP: this rank's ALTO-ordered shard (keys/vals, M nonzeros:
 * [bounds[r], bounds[r+1]) of balanced_bounds(M_total, world),
 * pkg/src/alto/partition.py:69-75) -> the factor-sized partial in `out`
 * (zeroed here) -> summed over the ranks. Local kernel: the ALTO
 * line-segment kernel when seg_bounds != NULL (alto_mttkrp_segment's tables
 * of this shard, acc_rows and privatize as there),
 * else the atomic key-stream kernel (alto_mttkrp_stream). owner_rows == 0:
 * in-place all-reduce, every rank ends with the full rows x ldo MTTKRP;
 * owner_rows != 0: `out` holds world * c rows (c = ceil(rows / world)) and
 * after an in-place reduce-scatter rank r's rows [r c, (r + 1) c) hold the
 * sum (the row owners of the sharded CP-ALS update). The reference result is
 * mttkrp(alto, factors, mode) (pkg/src/alto/kernels.py:284-303) up to the
 * order of the fp64 additions. */
int alto_mttkrp_sharded(const alto_layout_t *host_layout, const void *keys,
                        const double *vals, int64_t M,
                        const alto_factors_t *host_factors, int32_t mode,
                        double *out, int64_t ldo, int64_t rows,
                        const int64_t *seg_bounds, const int64_t *seg_lo,
                        int32_t L, int64_t acc_rows, int32_t privatize,
                        int32_t owner_rows, void *comm, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* ALTO_B200_H */
