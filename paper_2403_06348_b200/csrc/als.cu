// CP-ALS factor update on the device: one call per mode replaces the host
// round trip of pkg/src/alto/cpd/als.py:115-124 (v = hadamard_chain(grams,
// skip=n); a = solve_pseudo(mt, v); norms; a /= norms; grams[n] = gram(a))
// and pkg/src/alto/cpd/linalg.py:11-52, so a whole sweep can be queued (and
// captured in a CUDA graph) without a host sync per mode. Five short kernels:
//
//   1. als_chol_kernel (1 warp): V = Hadamard product of the other modes'
//      Grams (ascending mode order, as hadamard_chain), then its upper
//      Cholesky factor U (U^T U = V, dpotf2 order as scipy's cho_factor);
//      flags a non-PD or non-finite V.
//   2. als_solve_kernel: a sub-warp of RP lanes per row (lane = column):
//      U^T y = mt_i, U x = y with dtrsm's update order; x -> the factor.
//   3. als_gram_kernel: partial Grams G_b = A_b^T A_b of the unnormalised
//      rows over a few wide blocks (fixed-order partials).
//   4. als_final_kernel (1 block): G = sum of the partials in block order;
//      lambda = sqrt(diag G) (the column norms); grams[mode] = G / (s s^T)
//      with s = lambda (0 -> 1), i.e. the Gram of the normalised factor.
//   5. als_scale_kernel: a /= s.
// A non-PD V (the reference then takes the eigh pseudo-inverse) is only
// flagged: the driver restores the sweep's starting state and replays it on
// the host path. Non-finite MTTKRP output is flagged the same way.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "alto_common.cuh"

namespace alto {
namespace {

constexpr int kAlsThreads = 256;
constexpr int kGramBlocks = 64;
constexpr int kFlagNonfinite = 0;  // flags[0]: non-finite mt or V
constexpr int kFlagNotPd = 1;      // flags[1]: Cholesky failed

template <int RP>
__global__ void __launch_bounds__(32) als_chol_kernel(const double *__restrict__ grams, int nmodes, int mode,
                                                      int R, double *__restrict__ U, int *__restrict__ flags) {
  __shared__ double A[RP][RP + 1];
  const int lane = threadIdx.x;
  bool bad = false;
  for (int e = lane; e < R * R; e += 32) {
    const int i = e / R, j = e % R;
    double v = 1.0;
    bool first = true;
    for (int m = 0; m < nmodes; ++m) {
      if (m == mode) continue;
      const double g = grams[((int64_t)m * R + i) * R + j];
      v = first ? g : v * g;
      first = false;
    }
    A[i][j] = v;
    bad |= !isfinite(v);
  }
  __syncwarp();
  // upper Cholesky, column by column (dpotf2, uplo = 'U'): lane i < R owns
  // A(., i); ajj = A(j,j) - sum_{k<j} A(k,j)^2, A(j,i) = (A(j,i) - sum_k A(k,j) A(k,i)) / ajj
  bool fail = false;
  for (int j = 0; j < R; ++j) {
    double s = A[j][j];
    for (int k = 0; k < j; ++k) s -= A[k][j] * A[k][j];
    fail |= !(s > 0.0) || !isfinite(s);
    const double ajj = sqrt(s > 0.0 ? s : 1.0);
    if (lane > j && lane < R) {
      double t = A[j][lane];
      for (int k = 0; k < j; ++k) t -= A[k][j] * A[k][lane];
      A[j][lane] = t / ajj;
    }
    __syncwarp();
    if (lane == 0) A[j][j] = ajj;
    __syncwarp();
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&flags[kFlagNonfinite], 1);
  if (fail && lane == 0) atomicOr(&flags[kFlagNotPd], 1);
  for (int e = lane; e < R * R; e += 32) {
    const int i = e / R, j = e % R;
    U[e] = i <= j ? A[i][j] : 0.0;
  }
}

// a sub-warp of RP lanes per row (lane = column), 32/RP rows per warp: the
// substitutions run as R broadcast steps with dtrsm's update order
// (forward s_i -= U(k,i) y_k for ascending k; backward s_i -= U(i,k) x_k for
// descending k)
template <int RP>
__global__ void __launch_bounds__(kAlsThreads) als_solve_kernel(const double *__restrict__ mt, int64_t ldm,
                                                               double *__restrict__ a, int64_t lda, int64_t rows,
                                                               int R, const double *__restrict__ U,
                                                               int *__restrict__ flags) {
  constexpr int W = RP < 32 ? RP : 32;  // lanes per row
  __shared__ double Us[RP][RP + 1];
  const int tid = threadIdx.x, lane = tid & (W - 1);
  for (int e = tid; e < RP * RP; e += blockDim.x) {
    const int i = e / RP, j = e % RP;
    Us[i][j] = (i < R && j < R) ? U[i * R + j] : (i == j ? 1.0 : 0.0);
  }
  __syncthreads();
  const int64_t r = (blockIdx.x * (int64_t)blockDim.x + tid) / W;
  const bool col = lane < R;
  const bool ok = r < rows;
  const double ujj = col ? Us[lane][lane] : 1.0;
  double s = ok && col ? mt[r * ldm + lane] : 0.0;
  const bool bad = !isfinite(s);
  for (int j = 0; j < R; ++j) {  // U^T y = b
    if (lane == j) s = s / ujj;
    const double yj = __shfl_sync(0xffffffffu, s, j, W);
    if (lane > j && col) s -= Us[j][lane] * yj;
  }
  for (int j = R - 1; j >= 0; --j) {  // U x = y
    if (lane == j) s = s / ujj;
    const double xj = __shfl_sync(0xffffffffu, s, j, W);
    if (lane < j) s -= Us[lane][j] * xj;
  }
  if (ok && col) a[r * lda + lane] = s;
  if (__any_sync(0xffffffffu, bad) && (tid & 31) == 0) atomicOr(&flags[kFlagNonfinite], 1);
}

// partial Grams of the unnormalised rows; a few wide blocks so the final
// fixed-order reduction is short
template <int RP>
__global__ void __launch_bounds__(kAlsThreads) als_gram_kernel(const double *__restrict__ a, int64_t lda,
                                                              int64_t rows, int R,
                                                              double *__restrict__ gram_part) {
  constexpr int T = RP <= 16 ? 128 : 64;  // rows per tile
  constexpr int Q = (RP * RP + kAlsThreads - 1) / kAlsThreads;
  __shared__ double tile[T][RP + 1];
  const int tid = threadIdx.x;
  double g[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) g[q] = 0.0;
  for (int64_t t0 = blockIdx.x * (int64_t)T; t0 < rows; t0 += (int64_t)gridDim.x * T) {
    for (int e = tid; e < T * RP; e += kAlsThreads) {
      const int k = e / RP, j = e % RP;
      const int64_t r = t0 + k;
      tile[k][j] = (r < rows && j < R) ? a[r * lda + j] : 0.0;
    }
    __syncthreads();
    const int n = (int)(rows - t0 < T ? rows - t0 : T);
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int e = tid + q * kAlsThreads;
      if (e < RP * RP) {
        const int i = e / RP, j = e % RP;
        double acc = g[q];
        for (int k = 0; k < n; ++k) acc += tile[k][i] * tile[k][j];
        g[q] = acc;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int e = tid + q * kAlsThreads;
    if (e < RP * RP) gram_part[(int64_t)blockIdx.x * RP * RP + e] = g[q];
  }
}

template <int RP>
__global__ void __launch_bounds__(1024) als_final_kernel(const double *__restrict__ gram_part, int nparts, int R,
                                                         double *__restrict__ weights, double *__restrict__ inv,
                                                         double *__restrict__ gram) {
  __shared__ double G[RP][RP + 1];
  __shared__ double sc[RP];
  const int tid = threadIdx.x;
  for (int e = tid; e < RP * RP; e += blockDim.x) {
    double acc = 0.0;
    for (int p = 0; p < nparts; ++p) acc += gram_part[(int64_t)p * RP * RP + e];
    G[e / RP][e % RP] = acc;
  }
  __syncthreads();
  if (tid < R) {
    const double nrm = sqrt(G[tid][tid]);
    weights[tid] = nrm;
    sc[tid] = nrm == 0.0 ? 1.0 : nrm;
    inv[tid] = sc[tid];
  }
  __syncthreads();
  for (int e = tid; e < R * R; e += blockDim.x) {
    const int i = e / R, j = e % R;
    gram[e] = G[i][j] / (sc[i] * sc[j]);
  }
}

template <int RP>
__global__ void __launch_bounds__(kAlsThreads) als_scale_kernel(double *__restrict__ a, int64_t lda, int64_t rows,
                                                               int R, const double *__restrict__ sc) {
  __shared__ double s[RP];
  if (threadIdx.x < RP) s[threadIdx.x] = threadIdx.x < R ? sc[threadIdx.x] : 1.0;
  __syncthreads();
  const int64_t n = rows * R;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / R;
    const int j = (int)(e - r * R);
    a[r * lda + j] /= s[j];
  }
}

// sharded update (row blocks on several ranks): fixed-order sum of the
// partial Grams -> raw Gram R x R (summed across ranks by the caller) ...
template <int RP>
__global__ void __launch_bounds__(1024) als_gram_sum_kernel(const double *__restrict__ gram_part, int nparts,
                                                            int R, double *__restrict__ raw) {
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int i = e / R, j = e % R;
    double acc = 0.0;
    for (int p = 0; p < nparts; ++p) acc += gram_part[(int64_t)p * RP * RP + i * RP + j];
    raw[e] = acc;
  }
}

// ... then lambda = sqrt(diag G), the normalised Gram and the scale factors
template <int RP>
__global__ void __launch_bounds__(1024) als_final_raw_kernel(const double *__restrict__ raw, int R,
                                                             double *__restrict__ weights, double *__restrict__ inv,
                                                             double *__restrict__ gram) {
  __shared__ double sc[RP];
  const int tid = threadIdx.x;
  if (tid < R) {
    const double nrm = sqrt(raw[tid * R + tid]);
    weights[tid] = nrm;
    sc[tid] = nrm == 0.0 ? 1.0 : nrm;
    inv[tid] = sc[tid];
  }
  __syncthreads();
  for (int e = tid; e < R * R; e += blockDim.x) {
    const int i = e / R, j = e % R;
    gram[e] = raw[e] / (sc[i] * sc[j]);
  }
}

// Two-kernel form of steps 2-5 for the single-GPU sweep (the five-kernel
// form spent ~43 us per c2 mode, latency-bound; profiles/r02_*):
//  * als_solve_rows_kernel: one thread per row, the row in registers, the
//    substitutions with U from shared memory in dtrsm's update order (the
//    same operations, in the same order, as als_solve_kernel's lanes); the
//    block's rows then give one fixed-order partial Gram per block;
//  * als_norm_scale_kernel: every block sums the R diagonal partials in
//    block order (the column norms), scales its rows, and writes its share of
//    the normalised Gram (entry e by block e % grid, partials in order).
constexpr int kRowThreads = 128;

template <int RP>
__global__ void __launch_bounds__(kRowThreads) als_solve_rows_kernel(const double *__restrict__ mt, int64_t ldm,
                                                                    double *__restrict__ a, int64_t lda,
                                                                    int64_t rows, int R,
                                                                    const double *__restrict__ U,
                                                                    int *__restrict__ flags,
                                                                    double *__restrict__ gram_part) {
  __shared__ double Us[RP][RP + 1];
  __shared__ double tile[kRowThreads][RP + 1];
  const int tid = threadIdx.x;
  for (int e = tid; e < RP * RP; e += blockDim.x) {
    const int i = e / RP, j = e % RP;
    Us[i][j] = (i < R && j < R) ? U[i * R + j] : (i == j ? 1.0 : 0.0);
  }
  __syncthreads();
  const int64_t r = blockIdx.x * (int64_t)kRowThreads + tid;
  const bool ok = r < rows;
  double s[RP];
  bool bad = false;
#pragma unroll
  for (int j = 0; j < RP; ++j) {
    s[j] = (ok && j < R) ? mt[r * ldm + j] : 0.0;
    bad = bad || !isfinite(s[j]);
  }
#pragma unroll
  for (int j = 0; j < RP; ++j) {  // U^T y = b
    if (j < R) {
      s[j] = s[j] / Us[j][j];
#pragma unroll
      for (int i = j + 1; i < RP; ++i)
        if (i < R) s[i] -= Us[j][i] * s[j];
    }
  }
#pragma unroll
  for (int j = RP - 1; j >= 0; --j) {  // U x = y
    if (j < R) {
      s[j] = s[j] / Us[j][j];
#pragma unroll
      for (int i = 0; i < j; ++i) s[i] -= Us[i][j] * s[j];
    }
  }
#pragma unroll
  for (int j = 0; j < RP; ++j) {
    if (ok && j < R) a[r * lda + j] = s[j];
    tile[tid][j] = (ok && j < R) ? s[j] : 0.0;
  }
  if (__any_sync(0xffffffffu, bad) && (tid & 31) == 0) atomicOr(&flags[kFlagNonfinite], 1);
  __syncthreads();
  for (int e = tid; e < RP * RP; e += kRowThreads) {
    const int i = e / RP, j = e % RP;
    double acc = 0.0;
    for (int k = 0; k < kRowThreads; ++k) acc += tile[k][i] * tile[k][j];
    gram_part[(int64_t)blockIdx.x * RP * RP + e] = acc;
  }
}

template <int RP>
__global__ void __launch_bounds__(kAlsThreads) als_norm_scale_kernel(const double *__restrict__ gram_part,
                                                                    int nparts, int R, double *__restrict__ a,
                                                                    int64_t lda, int64_t rows,
                                                                    double *__restrict__ weights,
                                                                    double *__restrict__ gram) {
  constexpr int NCH = kAlsThreads / RP;
  __shared__ double red[NCH][RP];
  __shared__ double sc[RP];
  __shared__ double tsum[kAlsThreads];
  const int tid = threadIdx.x;
  {
    const int d = tid % RP, c = tid / RP;
    double acc = 0.0;
    if (d < R)
      for (int p = c; p < nparts; p += NCH) acc += gram_part[(int64_t)p * RP * RP + d * RP + d];
    red[c][d] = acc;
  }
  __syncthreads();
  if (tid < RP) {
    double acc = 0.0;
    for (int c = 0; c < NCH; ++c) acc += red[c][tid];
    const double nrm = sqrt(acc);
    sc[tid] = (tid < R && nrm != 0.0) ? nrm : 1.0;
    if (blockIdx.x == 0 && tid < R) weights[tid] = nrm;
  }
  __syncthreads();
  for (int e = blockIdx.x; e < R * R; e += gridDim.x) {
    const int i = e / R, j = e % R;
    double acc = 0.0;
    for (int p = tid; p < nparts; p += kAlsThreads) acc += gram_part[(int64_t)p * RP * RP + i * RP + j];
    tsum[tid] = acc;
    __syncthreads();
    for (int w = kAlsThreads / 2; w > 0; w >>= 1) {
      if (tid < w) tsum[tid] += tsum[tid + w];
      __syncthreads();
    }
    if (tid == 0) gram[e] = tsum[0] / (sc[i] * sc[j]);
    __syncthreads();
  }
  const int64_t n = rows * R;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + tid; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / R;
    const int j = (int)(e - r * R);
    a[r * lda + j] /= sc[j];
  }
}

int rows_blocks(int64_t rows) { return (int)((rows + kRowThreads - 1) / kRowThreads); }

int rp_for(int R) { return R <= 4 ? 4 : (R <= 8 ? 8 : (R <= 16 ? 16 : 32)); }

bool two_kernel_update() {
  static const int on = [] {
    const char *v = getenv("ALTO_B200_ALS_TWO_KERNEL");
    return (v == nullptr || *v == 0 || strcmp(v, "0") != 0) ? 1 : 0;
  }();
  return on != 0;
}

int gram_blocks(int64_t rows) {
  const int64_t b = (rows + 127) / 128;
  return (int)(b < 1 ? 1 : (b > kGramBlocks ? kGramBlocks : b));
}

template <int RP>
int als_update_rp(const double *mt, int64_t ldm, int64_t rows, int R, double *grams, int nmodes, int mode,
                  double *a, int64_t lda, double *weights, char *scratch, int *flags, bool do_chol,
                  cudaStream_t st) {
  constexpr int W = RP < 32 ? RP : 32;
  double *U = reinterpret_cast<double *>(scratch);
  double *inv = U + RP * RP;
  double *gpart = inv + RP;
  const int gb = gram_blocks(rows);
  if (do_chol) {
    als_chol_kernel<RP><<<1, 32, 0, st>>>(grams, nmodes, mode, R, U, flags);
    ALTO_LAUNCH_CHECK("als_chol_kernel");
  }
  if (two_kernel_update()) {
    const int nb = rows_blocks(rows);
    als_solve_rows_kernel<RP><<<nb, kRowThreads, 0, st>>>(mt, ldm, a, lda, rows, R, U, flags, gpart);
    ALTO_LAUNCH_CHECK("als_solve_rows_kernel");
    int cb = (int)((rows * R + kAlsThreads - 1) / kAlsThreads);
    if (cb > num_sms() * 2) cb = num_sms() * 2;
    if (cb < 1) cb = 1;
    als_norm_scale_kernel<RP><<<cb, kAlsThreads, 0, st>>>(gpart, nb, R, a, lda, rows, weights,
                                                          grams + (int64_t)mode * R * R);
    ALTO_LAUNCH_CHECK("als_norm_scale_kernel");
    return ALTO_OK;
  }
  (void)inv;
  const int64_t sb = (rows * W + kAlsThreads - 1) / kAlsThreads;
  als_solve_kernel<RP><<<(int)sb, kAlsThreads, 0, st>>>(mt, ldm, a, lda, rows, R, U, flags);
  ALTO_LAUNCH_CHECK("als_solve_kernel");
  als_gram_kernel<RP><<<gb, kAlsThreads, 0, st>>>(a, lda, rows, R, gpart);
  ALTO_LAUNCH_CHECK("als_gram_kernel");
  als_final_kernel<RP><<<1, RP * RP < 1024 ? RP * RP : 1024, 0, st>>>(gpart, gb, R, weights, inv,
                                                                      grams + (int64_t)mode * R * R);
  ALTO_LAUNCH_CHECK("als_final_kernel");
  int64_t cb = (rows * R + kAlsThreads - 1) / kAlsThreads;
  if (cb > (int64_t)num_sms() * 4) cb = (int64_t)num_sms() * 4;
  als_scale_kernel<RP><<<(int)cb, kAlsThreads, 0, st>>>(a, lda, rows, R, inv);
  ALTO_LAUNCH_CHECK("als_scale_kernel");
  return ALTO_OK;
}

template <int RP>
int als_solve_gram_rp(const double *mt, int64_t ldm, int64_t rows, int R, const double *grams, int nmodes,
                      int mode, double *a, int64_t lda, char *scratch, int *flags, bool do_chol, double *raw,
                      cudaStream_t st) {
  double *U = reinterpret_cast<double *>(scratch);
  double *inv = U + RP * RP;
  double *gpart = inv + RP;
  const int gb = gram_blocks(rows);
  constexpr int W = RP < 32 ? RP : 32;
  if (do_chol) {
    als_chol_kernel<RP><<<1, 32, 0, st>>>(grams, nmodes, mode, R, U, flags);
    ALTO_LAUNCH_CHECK("als_chol_kernel");
  }
  const int64_t sb = (rows * W + kAlsThreads - 1) / kAlsThreads;
  als_solve_kernel<RP><<<(int)sb, kAlsThreads, 0, st>>>(mt, ldm, a, lda, rows, R, U, flags);
  ALTO_LAUNCH_CHECK("als_solve_kernel");
  als_gram_kernel<RP><<<gb, kAlsThreads, 0, st>>>(a, lda, rows, R, gpart);
  ALTO_LAUNCH_CHECK("als_gram_kernel");
  als_gram_sum_kernel<RP><<<1, RP * RP < 1024 ? RP * RP : 1024, 0, st>>>(gpart, gb, R, raw);
  ALTO_LAUNCH_CHECK("als_gram_sum_kernel");
  return ALTO_OK;
}

template <int RP>
int als_normalize_rp(const double *raw, int R, double *grams, int mode, double *a, int64_t lda, int64_t rows,
                     double *weights, char *scratch, cudaStream_t st) {
  double *inv = reinterpret_cast<double *>(scratch) + RP * RP;
  als_final_raw_kernel<RP><<<1, RP * RP < 1024 ? RP * RP : 1024, 0, st>>>(raw, R, weights, inv,
                                                                          grams + (int64_t)mode * R * R);
  ALTO_LAUNCH_CHECK("als_final_raw_kernel");
  if (rows > 0) {
    int64_t cb = (rows * R + kAlsThreads - 1) / kAlsThreads;
    if (cb > (int64_t)num_sms() * 4) cb = (int64_t)num_sms() * 4;
    als_scale_kernel<RP><<<(int)cb, kAlsThreads, 0, st>>>(a, lda, rows, R, inv);
    ALTO_LAUNCH_CHECK("als_scale_kernel");
  }
  return ALTO_OK;
}

}  // namespace
}  // namespace alto

using namespace alto;

extern "C" {

int alto_als_update_scratch_bytes(int64_t rows, int32_t rank, size_t *host_bytes) {
  const int RP = rp_for(rank);
  int gb = gram_blocks(rows < 1 ? 1 : rows);
  if (gb < rows_blocks(rows < 1 ? 1 : rows)) gb = rows_blocks(rows < 1 ? 1 : rows);  // per-block partials
  *host_bytes = sizeof(double) * ((size_t)RP * RP + (size_t)RP + (size_t)gb * RP * RP) + 256;
  return ALTO_OK;
}

int alto_als_chol(const double *grams, int32_t nmodes, int32_t mode, int32_t rank, void *scratch,
                  size_t scratch_bytes, int32_t *flags, void *stream) {
  ALTO_REQUIRE(rank >= 1 && rank <= 32, ALTO_ERR_UNSUPPORTED, "device ALS update supports rank <= 32");
  ALTO_REQUIRE(mode >= 0 && mode < nmodes, ALTO_ERR_VALUE, "mode %d out of range", mode);
  const int RP = rp_for(rank);
  ALTO_REQUIRE(scratch_bytes >= sizeof(double) * (size_t)RP * RP, ALTO_ERR_VALUE, "ALS scratch too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double *U = static_cast<double *>(scratch);
  switch (RP) {
    case 4: als_chol_kernel<4><<<1, 32, 0, st>>>(grams, nmodes, mode, rank, U, flags); break;
    case 8: als_chol_kernel<8><<<1, 32, 0, st>>>(grams, nmodes, mode, rank, U, flags); break;
    case 16: als_chol_kernel<16><<<1, 32, 0, st>>>(grams, nmodes, mode, rank, U, flags); break;
    default: als_chol_kernel<32><<<1, 32, 0, st>>>(grams, nmodes, mode, rank, U, flags); break;
  }
  ALTO_LAUNCH_CHECK("als_chol_kernel");
  return ALTO_OK;
}

int alto_als_update_solve(const double *mt, int64_t ldm, int64_t rows, int32_t rank, double *grams,
                          int32_t nmodes, int32_t mode, double *a, int64_t lda, double *weights, void *scratch,
                          size_t scratch_bytes, int32_t *flags, int32_t do_chol, void *stream);

int alto_als_update(const double *mt, int64_t ldm, int64_t rows, int32_t rank, double *grams, int32_t nmodes,
                    int32_t mode, double *a, int64_t lda, double *weights, void *scratch, size_t scratch_bytes,
                    int32_t *flags, void *stream) {
  return alto_als_update_solve(mt, ldm, rows, rank, grams, nmodes, mode, a, lda, weights, scratch, scratch_bytes,
                               flags, 1, stream);
}

int alto_als_update_solve(const double *mt, int64_t ldm, int64_t rows, int32_t rank, double *grams,
                          int32_t nmodes, int32_t mode, double *a, int64_t lda, double *weights, void *scratch,
                          size_t scratch_bytes, int32_t *flags, int32_t do_chol, void *stream) {
  ALTO_REQUIRE(rank >= 1 && rank <= 32, ALTO_ERR_UNSUPPORTED, "device ALS update supports rank <= 32");
  ALTO_REQUIRE(mode >= 0 && mode < nmodes, ALTO_ERR_VALUE, "mode %d out of range", mode);
  ALTO_REQUIRE(rows >= 1, ALTO_ERR_VALUE, "empty factor");
  size_t need = 0;
  alto_als_update_scratch_bytes(rows, rank, &need);
  ALTO_REQUIRE(scratch_bytes >= need, ALTO_ERR_VALUE, "ALS scratch too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char *s = static_cast<char *>(scratch);
  const bool dc = do_chol != 0;
  switch (rp_for(rank)) {
    case 4: return als_update_rp<4>(mt, ldm, rows, rank, grams, nmodes, mode, a, lda, weights, s, flags, dc, st);
    case 8: return als_update_rp<8>(mt, ldm, rows, rank, grams, nmodes, mode, a, lda, weights, s, flags, dc, st);
    case 16:
      return als_update_rp<16>(mt, ldm, rows, rank, grams, nmodes, mode, a, lda, weights, s, flags, dc, st);
    default:
      return als_update_rp<32>(mt, ldm, rows, rank, grams, nmodes, mode, a, lda, weights, s, flags, dc, st);
  }
}

int alto_als_solve_gram(const double *mt, int64_t ldm, int64_t rows, int32_t rank, const double *grams,
                        int32_t nmodes, int32_t mode, double *a, int64_t lda, void *scratch, size_t scratch_bytes,
                        int32_t *flags, int32_t do_chol, double *gram_raw, void *stream) {
  ALTO_REQUIRE(rank >= 1 && rank <= 32, ALTO_ERR_UNSUPPORTED, "device ALS update supports rank <= 32");
  ALTO_REQUIRE(mode >= 0 && mode < nmodes, ALTO_ERR_VALUE, "mode %d out of range", mode);
  ALTO_REQUIRE(rows >= 1, ALTO_ERR_VALUE, "empty row block");
  size_t need = 0;
  alto_als_update_scratch_bytes(rows, rank, &need);
  ALTO_REQUIRE(scratch_bytes >= need, ALTO_ERR_VALUE, "ALS scratch too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char *s = static_cast<char *>(scratch);
  const bool dc = do_chol != 0;
  switch (rp_for(rank)) {
    case 4: return als_solve_gram_rp<4>(mt, ldm, rows, rank, grams, nmodes, mode, a, lda, s, flags, dc, gram_raw, st);
    case 8: return als_solve_gram_rp<8>(mt, ldm, rows, rank, grams, nmodes, mode, a, lda, s, flags, dc, gram_raw, st);
    case 16:
      return als_solve_gram_rp<16>(mt, ldm, rows, rank, grams, nmodes, mode, a, lda, s, flags, dc, gram_raw, st);
    default:
      return als_solve_gram_rp<32>(mt, ldm, rows, rank, grams, nmodes, mode, a, lda, s, flags, dc, gram_raw, st);
  }
}

int alto_als_normalize(const double *gram_raw, int32_t rank, double *grams, int32_t nmodes, int32_t mode, double *a,
                       int64_t lda, int64_t rows, double *weights, void *scratch, size_t scratch_bytes,
                       void *stream) {
  ALTO_REQUIRE(rank >= 1 && rank <= 32, ALTO_ERR_UNSUPPORTED, "device ALS update supports rank <= 32");
  ALTO_REQUIRE(mode >= 0 && mode < nmodes, ALTO_ERR_VALUE, "mode %d out of range", mode);
  const int RP = rp_for(rank);
  ALTO_REQUIRE(scratch_bytes >= sizeof(double) * ((size_t)RP * RP + RP), ALTO_ERR_VALUE, "ALS scratch too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char *s = static_cast<char *>(scratch);
  switch (RP) {
    case 4: return als_normalize_rp<4>(gram_raw, rank, grams, mode, a, lda, rows, weights, s, st);
    case 8: return als_normalize_rp<8>(gram_raw, rank, grams, mode, a, lda, rows, weights, s, st);
    case 16: return als_normalize_rp<16>(gram_raw, rank, grams, mode, a, lda, rows, weights, s, st);
    default: return als_normalize_rp<32>(gram_raw, rank, grams, mode, a, lda, rows, weights, s, st);
  }
}

}  // extern "C"
