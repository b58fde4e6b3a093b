// CP-APR support kernels on sm_100a: Khatri-Rao rows (PRE), the fused
// KKT / multiplicative-update epilogue, and the Poisson log-likelihood pass.
#include <math.h>
#include <string.h>

#include "run_kernels.cuh"

namespace alto {

// Pi[x][r] = prod_{m != mode, ascending} A_m[i_m, r]  (starts from 1.0 like
// np.ones(...) *= f[coords[:, m]] in pkg/src/alto/cpd/apr.py:107-111).
// One warp walks 32 nonzeros: lane q decodes key q, then the warp writes the
// 32 rows with lanes over columns.
__global__ void pi_kernel(const __grid_constant__ Layout L, const uint64_t *__restrict__ keys, int64_t M,
                          const __grid_constant__ Factors F, int mode, double *__restrict__ pi,
                          int64_t ldp) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int N = L.nmodes;
  const int R = F.rank;
  for (int64_t base = warp * 32; base < M; base += nwarps * 32) {
    const int64_t x = base + lane;
    Key k{0, 0};
    if (x < M) {
      k.w0 = keys[L.words * x];
      if (L.words == 2) k.w1 = keys[2 * x + 1];
    }
    const int cnt = (int)(M - base < 32 ? M - base : 32);
    for (int q = 0; q < cnt; ++q) {
      Key kb;
      kb.w0 = __shfl_sync(0xffffffffu, k.w0, q);
      kb.w1 = __shfl_sync(0xffffffffu, k.w1, q);
      for (int r = lane; r < R; r += 32) {
        double p = 1.0;
        for (int m = 0; m < N; ++m) {
          if (m == mode) continue;
          const int64_t i = (int64_t)decode_mode(L, m, kb);
          p = __dmul_rn(p, F.ptr[m][i * F.ld[m] + r]);
        }
        pi[(base + q) * ldp + r] = p;
      }
    }
  }
}

// kkt = max |min(b, 1 - phi)|; bits of a nonnegative double order like the
// double, so an unsigned max works. NaN is tracked separately.
__global__ void kkt_kernel(const double *__restrict__ b, int64_t ldb, const double *__restrict__ phi,
                           int64_t ldphi, int64_t rows, int rank, unsigned long long *__restrict__ kkt_bits,
                           int *__restrict__ nan_flag) {
  unsigned long long best = 0ull;
  bool nan = false;
  const int64_t total = rows * rank;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    // rows * rank < 2^31 for every realistic factor (checked by the caller)
    const uint32_t ue = (uint32_t)e, ur = (uint32_t)rank;
    const int64_t i = ue / ur;
    const int r = (int)(ue - (uint32_t)i * ur);
    const double bv = b[i * ldb + r];
    const double pv = phi[i * ldphi + r];
    const double t = __dsub_rn(1.0, pv);
    double m = bv < t ? bv : t;
    if (isnan(bv) || isnan(t)) nan = true;
    m = fabs(m);
    const unsigned long long bits = (unsigned long long)__double_as_longlong(m);
    best = bits > best ? bits : best;
  }
  for (int o = 16; o; o >>= 1) {
    const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
    best = other > best ? other : best;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(kkt_bits, best);
  if (__any_sync(0xffffffffu, nan) && (threadIdx.x & 31) == 0) atomicOr(nan_flag, 1);
}

// b *= phi when the device-side decision says so (apply < 0: iff kkt >= tau
// or kkt is NaN, mirroring `if kkt < tau: break` in pkg/src/alto/cpd/apr.py:302).
__global__ void apply_kernel(double *__restrict__ b, int64_t ldb, const double *__restrict__ phi,
                             int64_t ldphi, int64_t rows, int rank, double tau, int apply,
                             const unsigned long long *__restrict__ kkt_bits,
                             const int *__restrict__ nan_flag, int *__restrict__ nonfinite) {
  bool go;
  if (apply >= 0) {
    go = apply != 0;
  } else {
    const double kkt = __longlong_as_double((long long)*kkt_bits);
    go = (*nan_flag != 0) || !(kkt < tau);
  }
  if (!go) return;
  bool bad = false;
  const int64_t total = rows * rank;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    // rows * rank < 2^31 for every realistic factor (checked by the caller)
    const uint32_t ue = (uint32_t)e, ur = (uint32_t)rank;
    const int64_t i = ue / ur;
    const int r = (int)(ue - (uint32_t)i * ur);
    const double v = __dmul_rn(b[i * ldb + r], phi[i * ldphi + r]);
    b[i * ldb + r] = v;
    if (!isfinite(v)) bad = true;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1);
}

// ---- device-driven inner loop ---------------------------------------------
// The reference's inner loop (pkg/src/alto/cpd/apr.py:290-310) decides after
// every Phi whether to stop (kkt < tau). Here the decision stays on the
// device: the host enqueues all max_inner iterations at once, every kernel of
// an iteration returns immediately once `done` is set, and the host reads the
// outcome (iterations used, last KKT, first non-finite update) once per mode.
constexpr int kMaxInner = 1024;
struct InnerState {
  int32_t done;            // the loop broke (kkt < tau) or an update went non-finite
  int32_t nonfinite_iter;  // 1 + first iteration whose update was non-finite (0: none)
  int32_t used;            // Phi evaluations performed
  int32_t pad;
  unsigned long long kbits[kMaxInner];
  int32_t nan[kMaxInner];
  double kkt[kMaxInner];
};

__global__ void inner_kkt_kernel(const double *__restrict__ b, int64_t ldb, const double *__restrict__ phi,
                                 int64_t ldphi, int64_t rows, int rank, InnerState *s, int it) {
  if (*reinterpret_cast<volatile const int32_t *>(&s->done)) return;
  unsigned long long best = 0ull;
  bool nan = false;
  const int64_t total = rows * rank;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t ue = (uint32_t)e, ur = (uint32_t)rank;
    const int64_t i = ue / ur;
    const int r = (int)(ue - (uint32_t)i * ur);
    const double bv = b[i * ldb + r];
    const double t = __dsub_rn(1.0, phi[i * ldphi + r]);
    double m = bv < t ? bv : t;
    if (isnan(bv) || isnan(t)) nan = true;
    m = fabs(m);
    const unsigned long long bits = (unsigned long long)__double_as_longlong(m);
    best = bits > best ? bits : best;
  }
  for (int o = 16; o; o >>= 1) {
    const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
    best = other > best ? other : best;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(&s->kbits[it], best);
  if (__any_sync(0xffffffffu, nan) && (threadIdx.x & 31) == 0) atomicOr(&s->nan[it], 1);
}

__global__ void inner_apply_kernel(double *__restrict__ b, int64_t ldb, const double *__restrict__ phi,
                                   int64_t ldphi, int64_t rows, int rank, double tau, InnerState *s, int it) {
  if (*reinterpret_cast<volatile const int32_t *>(&s->done)) return;
  const double kkt = __longlong_as_double((long long)s->kbits[it]);
  const bool nan = s->nan[it] != 0;
  const bool go = nan || !(kkt < tau);  // `if kkt < tau: break` (NaN continues)
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    s->used = it + 1;
    s->kkt[it] = nan ? (double)NAN : kkt;
    if (!go) s->done = 1;  // other blocks either see it or have nothing to do
  }
  if (!go) return;
  bool bad = false;
  const int64_t total = rows * rank;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t ue = (uint32_t)e, ur = (uint32_t)rank;
    const int64_t i = ue / ur;
    const int r = (int)(ue - (uint32_t)i * ur);
    const double v = __dmul_rn(b[i * ldb + r], phi[i * ldphi + r]);
    b[i * ldb + r] = v;
    if (!isfinite(v)) bad = true;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) {
    atomicCAS(&s->nonfinite_iter, 0, it + 1);
    s->done = 1;  // the host raises NumericalError
  }
}

__global__ void zero_if_kernel(double *__restrict__ out, int64_t n, const InnerState *s) {
  if (*reinterpret_cast<volatile const int32_t *>(&s->done)) return;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = 0.0;
}

// Poisson log-likelihood data term: sum_x v_x log(sum_r lambda_r prod_n A_n[i_n, r]).
// Fixed grid + fixed-order reductions => deterministic.
constexpr int kLoglikBlocks = 148 * 4;

__global__ void loglik_kernel(const __grid_constant__ Layout L, const uint64_t *__restrict__ keys,
                              const double *__restrict__ vals, int64_t M,
                              const __grid_constant__ Factors F, const double *__restrict__ lambda,
                              double *__restrict__ partials) {
  __shared__ double warp_sums[8];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int N = L.nmodes;
  const int R = F.rank;
  double local = 0.0;
  for (int64_t base = warp * 32; base < M; base += nwarps * 32) {
    const int64_t x = base + lane;
    Key k{0, 0};
    double v = 0.0;
    if (x < M) {
      k.w0 = keys[L.words * x];
      if (L.words == 2) k.w1 = keys[2 * x + 1];
      v = vals[x];
    }
    const int cnt = (int)(M - base < 32 ? M - base : 32);
    for (int q = 0; q < cnt; ++q) {
      Key kb;
      kb.w0 = __shfl_sync(0xffffffffu, k.w0, q);
      kb.w1 = __shfl_sync(0xffffffffu, k.w1, q);
      const double vq = __shfl_sync(0xffffffffu, v, q);
      double t = 0.0;
      for (int r = lane; r < R; r += 32) {
        double p = 1.0;
        for (int m = 0; m < N; ++m) {
          const int64_t i = (int64_t)decode_mode(L, m, kb);
          p = __dmul_rn(p, F.ptr[m][i * F.ld[m] + r]);
        }
        t = fma(p, lambda[r], t);
      }
      for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (lane == 0) local += vq * log(t);
    }
  }
  if (lane == 0) warp_sums[wid] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += warp_sums[w];
    partials[blockIdx.x] = s;
  }
}

// Fast log-likelihood pass: the run_kernel work mapping (group of G lanes per
// nonzero, kVec columns per lane, in-register decode, batched gathers of all
// N factor rows), mhat = sum_r lambda_r prod_n A_n[i_n, r] reduced across the
// group, v * log(mhat) summed per group in stream order, then per block in a
// fixed order => deterministic for a fixed segment count.
template <int NM, int G, int KW>
__global__ void __launch_bounds__(256, 2)
    loglik_groups_kernel(const __grid_constant__ RunArgs a, const double *__restrict__ lambda,
                         double *__restrict__ partials) {
  constexpr int VEC = kVec;
  constexpr int U = G < RUN_U ? G : RUN_U;
  __shared__ double warp_sums[8];
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int gbase = lane & ~(G - 1);
  const int64_t seg = gtid / G;
  const bool seg_ok = seg < a.nseg;
  const int64_t s0 = seg_ok ? seg_begin(seg, a.M, a.nseg) : a.M;
  const int64_t s1 = seg_ok ? seg_begin(seg + 1, a.M, a.nseg) : a.M;
  const int colv = gl * VEC;
  const bool lane_active = colv < a.rank;
  const int colld = lane_active ? colv : 0;
  double lam[VEC];
#pragma unroll
  for (int q = 0; q < VEC; ++q) lam[q] = (colv + q < a.rank) ? lambda[colv + q] : 0.0;
  double local = 0.0;
  int nch = (int)((s1 - s0 + G - 1) / G);
#pragma unroll
  for (int o = 16; o; o >>= 1) nch = max(nch, __shfl_xor_sync(0xffffffffu, nch, o));
  for (int ch = 0; ch < nch; ++ch) {
    const int64_t base = s0 + (int64_t)ch * G;
    Key k{0, 0};
    double val = 0.0;
    if (base + gl < s1) {
      k = load_key_stream<KW>(a.keys, base + gl);
      val = ld_stream_f64(a.vals + base + gl);
    }
    uint32_t c[NM];
#pragma unroll
    for (int m = 0; m < NM; ++m) c[m] = (uint32_t)decode_fast<KW>(a.L, m, k);
    const int64_t rem = s1 - base;
    const int cnt = rem <= 0 ? 0 : (rem < (int64_t)G ? (int)rem : G);
#pragma unroll
    for (int ib = 0; ib < G; ib += U) {
      double f[NM][U][VEC];
#pragma unroll
      for (int m = 0; m < NM; ++m) {
        const double *fm = a.F.ptr[m] + colld;
        const uint32_t ldm = (uint32_t)a.F.ld[m];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t idx = __shfl_sync(0xffffffffu, c[m], gbase + ib + u);
          load_row<VEC>(fm + (uint64_t)idx * ldm, true, f[m][u]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double v = __shfl_sync(0xffffffffu, val, gbase + ib + u);
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < VEC; ++q) {
          double p = f[0][u][q];
#pragma unroll
          for (int m = 1; m < NM; ++m) p = __dmul_rn(p, f[m][u][q]);
          t = fma(p, lam[q], t);
        }
#pragma unroll
        for (int o = G / 2; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (gl == 0 && ib + u < cnt) local += v * log(t);
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if (lane == 0) warp_sums[threadIdx.x >> 5] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += warp_sums[w];
    partials[blockIdx.x] = s;
  }
}

__global__ void sum_partials_kernel(const double *__restrict__ partials, int n, double *__restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += partials[i];
    *out = s;
  }
}

static int64_t loglik_segments(int64_t M) { return M < 512 ? 1 : (M + 511) / 512; }

static int loglik_group_lanes(int rank) {
  int g = 1;
  while (g * kVec < rank) g *= 2;
  return g;
}

template <int NM, int KW>
static int launch_loglik_groups(const RunArgs &a, int g, int grid, const double *lambda, double *partials,
                                cudaStream_t st) {
  switch (g) {
    case 1: loglik_groups_kernel<NM, 1, KW><<<grid, 256, 0, st>>>(a, lambda, partials); break;
    case 2: loglik_groups_kernel<NM, 2, KW><<<grid, 256, 0, st>>>(a, lambda, partials); break;
    case 4: loglik_groups_kernel<NM, 4, KW><<<grid, 256, 0, st>>>(a, lambda, partials); break;
    default: loglik_groups_kernel<NM, 8, KW><<<grid, 256, 0, st>>>(a, lambda, partials); break;
  }
  ALTO_LAUNCH_CHECK("loglik_groups_kernel");
  return ALTO_OK;
}

}  // namespace alto

using namespace alto;

extern "C" {

int alto_pi(const alto_layout_t *host_layout, const void *keys, int64_t M,
            const alto_factors_t *host_factors, int32_t mode, double *pi, int64_t ldp, void *stream) {
  int rc = check_layout(host_layout);
  if (rc) return rc;
  rc = check_factors(host_layout, host_factors);
  if (rc) return rc;
  ALTO_REQUIRE(mode >= 0 && mode < host_layout->nmodes, ALTO_ERR_VALUE, "mode %d out of range", mode);
  if (M <= 0) return ALTO_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t blocks = ceil_div(M, 256);
  if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
  pi_kernel<<<(int)blocks, 256, 0, st>>>(to_device_layout(host_layout), static_cast<const uint64_t *>(keys),
                                        M, to_device_factors(host_factors), mode, pi, ldp);
  ALTO_LAUNCH_CHECK("pi_kernel");
  return ALTO_OK;
}

int alto_apr_update(double *b, int64_t ldb, const double *phi, int64_t ldphi, int64_t rows,
                    int32_t rank, double tau, int32_t apply, double *host_out, void *stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  struct Flags {
    unsigned long long kkt;
    int nan;
    int nonfinite;
  };
  ALTO_REQUIRE(rows * (int64_t)rank < (1ll << 31), ALTO_ERR_UNSUPPORTED, "factor too large for apr_update");
  void *dflag = nullptr, *hflag = nullptr;
  int rc = flag_scratch(&dflag, &hflag);
  if (rc) return rc;
  Flags *f = static_cast<Flags *>(dflag);
  ALTO_CUDA(cudaMemsetAsync(f, 0, sizeof(Flags), st));
  const int64_t total = rows * rank;
  int64_t blocks = ceil_div(total, 256);
  if (blocks > (int64_t)num_sms() * 4) blocks = (int64_t)num_sms() * 4;
  if (blocks < 1) blocks = 1;
  kkt_kernel<<<(int)blocks, 256, 0, st>>>(b, ldb, phi, ldphi, rows, rank, &f->kkt, &f->nan);
  ALTO_LAUNCH_CHECK("kkt_kernel");
  apply_kernel<<<(int)blocks, 256, 0, st>>>(b, ldb, phi, ldphi, rows, rank, tau, apply, &f->kkt, &f->nan,
                                            &f->nonfinite);
  ALTO_LAUNCH_CHECK("apply_kernel");
  ALTO_CUDA(cudaMemcpyAsync(hflag, f, sizeof(Flags), cudaMemcpyDeviceToHost, st));
  ALTO_CUDA(cudaStreamSynchronize(st));
  const Flags h = *static_cast<const Flags *>(hflag);
  double kkt;
  memcpy(&kkt, &h.kkt, sizeof kkt);
  host_out[0] = h.nan ? NAN : kkt;
  host_out[1] = h.nonfinite ? 1.0 : 0.0;
  return ALTO_OK;
}

int alto_apr_inner_state_bytes(int32_t max_inner, size_t *host_bytes) {
  ALTO_REQUIRE(max_inner >= 1 && max_inner <= kMaxInner, ALTO_ERR_UNSUPPORTED,
               "device-driven inner loop supports 1..%d iterations", kMaxInner);
  *host_bytes = sizeof(InnerState);
  return ALTO_OK;
}

int alto_apr_inner_kkt_offset(size_t *host_offset) {
  *host_offset = offsetof(InnerState, kkt);
  return ALTO_OK;
}

int alto_apr_inner_reset(void *state, void *stream) {
  ALTO_CUDA(cudaMemsetAsync(state, 0, sizeof(InnerState), static_cast<cudaStream_t>(stream)));
  return ALTO_OK;
}

int alto_zero_if(double *out, int64_t ld, int64_t rows, const void *state, void *stream) {
  const int64_t n = ld * rows;
  if (n <= 0) return ALTO_OK;
  int64_t blocks = ceil_div(n, 256);
  if (blocks > (int64_t)num_sms() * 4) blocks = (int64_t)num_sms() * 4;
  zero_if_kernel<<<(int)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      out, n, static_cast<const InnerState *>(state));
  ALTO_LAUNCH_CHECK("zero_if_kernel");
  return ALTO_OK;
}

__global__ void copy_if_kernel(const double *__restrict__ src, double *__restrict__ dst, int64_t n,
                               const InnerState *s) {
  if (*reinterpret_cast<volatile const int32_t *>(&s->done)) return;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = src[e];
}

int alto_copy_if(const double *src, double *dst, int64_t n, const void *state, void *stream) {
  if (n <= 0) return ALTO_OK;
  int64_t blocks = ceil_div(n, 256);
  if (blocks > (int64_t)num_sms() * 4) blocks = (int64_t)num_sms() * 4;
  copy_if_kernel<<<(int)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      src, dst, n, static_cast<const InnerState *>(state));
  ALTO_LAUNCH_CHECK("copy_if_kernel");
  return ALTO_OK;
}

int alto_apr_inner_step(double *b, int64_t ldb, const double *phi, int64_t ldphi, int64_t rows, int32_t rank,
                        double tau, int32_t iter, void *state, void *stream) {
  ALTO_REQUIRE(rows * (int64_t)rank < (1ll << 31), ALTO_ERR_UNSUPPORTED, "factor too large for apr_update");
  ALTO_REQUIRE(iter >= 0 && iter < kMaxInner, ALTO_ERR_VALUE, "inner iteration %d out of range", iter);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  InnerState *s = static_cast<InnerState *>(state);
  int64_t blocks = ceil_div(rows * rank, 256);
  if (blocks > (int64_t)num_sms() * 4) blocks = (int64_t)num_sms() * 4;
  if (blocks < 1) blocks = 1;
  inner_kkt_kernel<<<(int)blocks, 256, 0, st>>>(b, ldb, phi, ldphi, rows, rank, s, iter);
  ALTO_LAUNCH_CHECK("inner_kkt_kernel");
  inner_apply_kernel<<<(int)blocks, 256, 0, st>>>(b, ldb, phi, ldphi, rows, rank, tau, s, iter);
  ALTO_LAUNCH_CHECK("inner_apply_kernel");
  return ALTO_OK;
}

int alto_apr_inner_result(const void *state, int32_t *host_used, int32_t *host_nonfinite_iter,
                          double *host_kkt, void *stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  void *dflag = nullptr, *hflag = nullptr;
  int rc = flag_scratch(&dflag, &hflag);
  if (rc) return rc;
  const InnerState *s = static_cast<const InnerState *>(state);
  int32_t head[4];
  ALTO_CUDA(cudaMemcpyAsync(hflag, s, sizeof head, cudaMemcpyDeviceToHost, st));
  ALTO_CUDA(cudaStreamSynchronize(st));
  memcpy(head, hflag, sizeof head);
  *host_used = head[2];
  *host_nonfinite_iter = head[1];
  *host_kkt = NAN;
  if (head[2] > 0) {
    ALTO_CUDA(cudaMemcpyAsync(hflag, &s->kkt[head[2] - 1], sizeof(double), cudaMemcpyDeviceToHost, st));
    ALTO_CUDA(cudaStreamSynchronize(st));
    memcpy(host_kkt, hflag, sizeof(double));
  }
  return ALTO_OK;
}

int alto_loglik_partials(int64_t M, int32_t *host_count) {
  const int64_t fast_blocks = ceil_div(loglik_segments(M) * 8, 256) + 1;
  *host_count = (int32_t)((fast_blocks > kLoglikBlocks ? fast_blocks : kLoglikBlocks) + 1);
  return ALTO_OK;
}

int alto_loglik(const alto_layout_t *host_layout, const void *keys, const double *vals, int64_t M,
                const alto_factors_t *host_factors, const double *lambda, double *partials,
                double *host_sum, void *stream) {
  int rc = check_layout(host_layout);
  if (rc) return rc;
  rc = check_factors(host_layout, host_factors);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int N = host_layout->nmodes;
  const int R = host_factors->rank;
  int nblocks = kLoglikBlocks;
  bool fast = M > 0 && R <= kMaxRankChunk && (N == 3 || N == 4 || N == 5);
  for (int n = 0; n < N && fast; ++n) fast = host_layout->dims[n] <= 0xffffffffll;
  if (fast) {
    RunArgs a;
    memset(&a, 0, sizeof a);
    a.L = to_device_layout(host_layout);
    a.F = to_device_factors(host_factors);
    a.keys = static_cast<const uint64_t *>(keys);
    a.vals = vals;
    a.M = M;
    a.rank = R;
    a.full_rank = R;
    a.nseg = loglik_segments(M);
    const int g = loglik_group_lanes(R);
    nblocks = (int)ceil_div(a.nseg * g, 256);
    const bool w2 = host_layout->word_bits == 128;
    if (N == 3) rc = w2 ? launch_loglik_groups<3, 2>(a, g, nblocks, lambda, partials, st)
                        : launch_loglik_groups<3, 1>(a, g, nblocks, lambda, partials, st);
    else if (N == 4) rc = w2 ? launch_loglik_groups<4, 2>(a, g, nblocks, lambda, partials, st)
                             : launch_loglik_groups<4, 1>(a, g, nblocks, lambda, partials, st);
    else rc = w2 ? launch_loglik_groups<5, 2>(a, g, nblocks, lambda, partials, st)
                 : launch_loglik_groups<5, 1>(a, g, nblocks, lambda, partials, st);
    if (rc) return rc;
  } else {
    loglik_kernel<<<kLoglikBlocks, 256, 0, st>>>(to_device_layout(host_layout),
                                                 static_cast<const uint64_t *>(keys), vals, M,
                                                 to_device_factors(host_factors), lambda, partials);
    ALTO_LAUNCH_CHECK("loglik_kernel");
  }
  int32_t count = 0;
  alto_loglik_partials(M, &count);
  double *total = partials + (count - 1);
  sum_partials_kernel<<<1, 32, 0, st>>>(partials, nblocks, total);
  ALTO_LAUNCH_CHECK("sum_partials_kernel");
  if (host_sum) {
    ALTO_CUDA(cudaMemcpyAsync(host_sum, total, sizeof(double), cudaMemcpyDeviceToHost, st));
    ALTO_CUDA(cudaStreamSynchronize(st));
  }
  return ALTO_OK;
}

}  // extern "C"
