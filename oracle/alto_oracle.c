/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY. Never linked into or called by the
 * product path (paper_2403_06348_b200/). Used by tests/, by
 * __graft_entry__.smoke() as the checker, and by bench.py's cpu_baseline /
 * --impl reference leg as the timed CPU port of the reference.
 *
 * Plain-C restatement of the reference's compiled inner loops
 * (pkg/src/alto/_jit.py), same operation order and IEEE semantics as numba
 * without fastmath (compile with -ffp-contract=off): results are
 * bit-identical to the reference kernels for the same inputs.
 *
 *   alto_o_mttkrp_block        <- _jit.mttkrp_block        (_jit.py:16-30)
 *   alto_o_mttkrp_block_split  <- _jit.mttkrp_block_split  (_jit.py:33-50)
 *   alto_o_pull_reduce         <- _jit.pull_reduce         (_jit.py:53-64)
 *   alto_o_phi_block           <- _jit.phi_block           (_jit.py:67-102)
 *   alto_o_phi_block_split     <- _jit.phi_block_split     (_jit.py:105-137)
 *
 * Plus OpenMP drivers that restate the reference's thread-pool fan-out of
 * the recursive strategy (pkg/src/alto/kernels.py:187-210): segments in
 * parallel into private buffers, then row blocks of the pull reduction.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

void alto_o_mttkrp_block(const int64_t *coords, int64_t ncols, const double *vals,
                         const double *fstack, const int64_t *offs, int64_t nmodes,
                         int64_t rank, int64_t mode, int64_t start, int64_t stop, double *out,
                         int64_t row_base) {
  for (int64_t x = start; x < stop; ++x) {
    const int64_t *c = coords + x * ncols;
    double *o = out + (c[mode] - row_base) * rank;
    const double v = vals[x];
    for (int64_t r = 0; r < rank; ++r) {
      double p = v;
      for (int64_t m = 0; m < nmodes; ++m)
        if (m != mode) p *= fstack[(offs[m] + c[m]) * rank + r];
      o[r] += p;
    }
  }
}

void alto_o_mttkrp_block_split(const int64_t *coords, int64_t ncols, const double *vals,
                               const double *fstack, const int64_t *offs, int64_t nmodes,
                               int64_t rank, int64_t mode, int64_t start, int64_t stop,
                               double *out, const int64_t *slots, double *bbuf) {
  for (int64_t x = start; x < stop; ++x) {
    const int64_t *c = coords + x * ncols;
    const int64_t row = c[mode];
    const int64_t s = slots[row];
    double *o = s >= 0 ? bbuf + s * rank : out + row * rank;
    const double v = vals[x];
    for (int64_t r = 0; r < rank; ++r) {
      double p = v;
      for (int64_t m = 0; m < nmodes; ++m)
        if (m != mode) p *= fstack[(offs[m] + c[m]) * rank + r];
      o[r] += p;
    }
  }
}

void alto_o_pull_reduce(const double *temps, const int64_t *seg_offs, const int64_t *lo,
                        const int64_t *hi, int64_t nseg, double *out, int64_t rank,
                        int64_t row_start, int64_t row_stop) {
  for (int64_t b = row_start; b < row_stop; ++b)
    for (int64_t l = 0; l < nseg; ++l)
      if (lo[l] <= b && b <= hi[l]) {
        const double *t = temps + seg_offs[l] + (b - lo[l]) * rank;
        for (int64_t r = 0; r < rank; ++r) out[b * rank + r] += t[r];
      }
}

static void phi_one(const int64_t *c, double v, const double *fstack, const int64_t *offs,
                    int64_t nmodes, int64_t rank, int64_t mode, const double *scaled,
                    const double *krp_row, double eps, double *krp, double *o) {
  const int64_t row = c[mode];
  if (krp_row) {
    for (int64_t r = 0; r < rank; ++r) krp[r] = krp_row[r];
  } else {
    for (int64_t r = 0; r < rank; ++r) krp[r] = 1.0;
    for (int64_t m = 0; m < nmodes; ++m) {
      if (m == mode) continue;
      const double *f = fstack + (offs[m] + c[m]) * rank;
      for (int64_t r = 0; r < rank; ++r) krp[r] *= f[r];
    }
  }
  double d = 0.0;
  for (int64_t r = 0; r < rank; ++r) d += scaled[row * rank + r] * krp[r];
  if (d < eps) d = eps;
  const double w = v / d;
  for (int64_t r = 0; r < rank; ++r) o[r] += w * krp[r];
}

void alto_o_phi_block(const int64_t *coords, int64_t ncols, const double *vals,
                      const double *fstack, const int64_t *offs, int64_t nmodes, int64_t rank,
                      const double *scaled, const double *krp_rows, int64_t use_pre, double eps,
                      int64_t mode, int64_t start, int64_t stop, double *out, int64_t row_base) {
  double *krp = (double *)malloc(sizeof(double) * (size_t)(rank > 0 ? rank : 1));
  for (int64_t x = start; x < stop; ++x) {
    const int64_t *c = coords + x * ncols;
    phi_one(c, vals[x], fstack, offs, nmodes, rank, mode, scaled,
            use_pre ? krp_rows + x * rank : NULL, eps, krp, out + (c[mode] - row_base) * rank);
  }
  free(krp);
}

void alto_o_phi_block_split(const int64_t *coords, int64_t ncols, const double *vals,
                            const double *fstack, const int64_t *offs, int64_t nmodes,
                            int64_t rank, const double *scaled, const double *krp_rows,
                            int64_t use_pre, double eps, int64_t mode, int64_t start,
                            int64_t stop, double *out, const int64_t *slots, double *bbuf) {
  double *krp = (double *)malloc(sizeof(double) * (size_t)(rank > 0 ? rank : 1));
  for (int64_t x = start; x < stop; ++x) {
    const int64_t *c = coords + x * ncols;
    const int64_t s = slots[c[mode]];
    double *o = s >= 0 ? bbuf + s * rank : out + c[mode] * rank;
    phi_one(c, vals[x], fstack, offs, nmodes, rank, mode, scaled,
            use_pre ? krp_rows + x * rank : NULL, eps, krp, o);
  }
  free(krp);
}

/* Recursive strategy, thread-parallel (restates _accumulate_segments +
 * _reduce_rows, pkg/src/alto/kernels.py:187-210). phi != 0 selects the Phi
 * block. temps must be zeroed, sized sum(widths) * rank. */
void alto_o_recursive(const int64_t *coords, int64_t ncols, const double *vals,
                      const double *fstack, const int64_t *offs, int64_t nmodes, int64_t rank,
                      int64_t mode, const int64_t *bounds, const int64_t *lo, const int64_t *hi,
                      const int64_t *seg_offs, int64_t nseg, double *temps, double *out,
                      int64_t out_rows, int64_t phi, const double *scaled,
                      const double *krp_rows, int64_t use_pre, double eps, int64_t threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads((int)threads);
#endif
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t l = 0; l < nseg; ++l) {
    if (phi)
      alto_o_phi_block(coords, ncols, vals, fstack, offs, nmodes, rank, scaled, krp_rows, use_pre,
                       eps, mode, bounds[l], bounds[l + 1], temps + seg_offs[l], lo[l]);
    else
      alto_o_mttkrp_block(coords, ncols, vals, fstack, offs, nmodes, rank, mode, bounds[l],
                          bounds[l + 1], temps + seg_offs[l], lo[l]);
  }
  int64_t nblk = threads > 0 ? threads : 1;
  if (nblk > out_rows) nblk = out_rows > 0 ? out_rows : 1;
#pragma omp parallel for schedule(static, 1)
  for (int64_t i = 0; i < nblk; ++i) {
    const int64_t base = out_rows / nblk, extra = out_rows % nblk;
    const int64_t a = i * base + (i < extra ? i : extra);
    const int64_t b = a + base + (i < extra ? 1 : 0);
    alto_o_pull_reduce(temps, seg_offs, lo, hi, nseg, out, rank, a, b);
  }
}
