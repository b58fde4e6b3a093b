// Fiber kernels: MTTKRP / Phi over a mode-ordered view whose rows are
// sub-sorted by a second ("fiber") mode a, so that consecutive nonzeros of a
// row share the same a-index in runs (fibers).
//
//   MTTKRP:  out[i] += sum_j A_a[j] o ( sum_{x in fiber (i,j)} v_x prod_{rest} F_m[i_m] )
//   Phi:     krp_x = A_a[j] o prod_{rest} F_m[i_m]   (A_a[j] kept in registers per fiber,
//            the scaled row B[i] kept in registers per row run)
//
// Compared with run_kernel the A_a row is gathered once per fiber instead of
// once per nonzero (and for MTTKRP multiplied once per fiber), which removes
// most of the L1 traffic on Zipf-skewed tensors where fibers are long.
// Register row runs, segment edges and the warp-uniform control flow are the
// same as run_kernel (fast path: edge runs are reduced with fp64 atomics).
// Summation order differs from the reference's, so this is a fast-path
// kernel only (<= 1e-12 relative on the parity suite); exact parity uses
// run_kernel / the exact segment kernels.
#pragma once

#include "run_kernels.cuh"

namespace alto {

template <int NM, int G, int KW, bool PHI>
__global__ void __launch_bounds__(256, 2) fiber_kernel(const __grid_constant__ RunArgs a) {
  constexpr int VEC = kVec;
  constexpr int UB = 2;  // fiber/row state lives in registers: keep batches small
  constexpr int U = G < UB ? G : UB;
  constexpr int NR = NM - 2;  // "rest" modes multiplied per nonzero
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int gbase = lane & ~(G - 1);
  const int64_t seg = gtid / G;
  const bool seg_ok = seg < a.nseg;
  const int64_t s0 = seg_ok ? seg_begin(seg, a.M, a.nseg) : a.M;
  const int64_t s1 = seg_ok ? seg_begin(seg + 1, a.M, a.nseg) : a.M;
  const int mode = a.mode;
  const int fm = a.fiber_mode;

  const int colv = gl * VEC;
  bool colok[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) colok[v] = colv + v < a.rank;
  const bool lane_active = colok[0];
  const int colld = lane_active ? colv : 0;

  // rest modes in ascending order: the j-th mode of 0..NM-1 once mode and
  // the fiber mode are removed (selects only: no dynamic register indexing)
  int rest[NR > 0 ? NR : 1];
  {
    const int lo = mode < fm ? mode : fm, hi = mode < fm ? fm : mode;
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      int r = j;
      if (r >= lo) ++r;
      if (r >= hi) ++r;
      rest[j] = r;
    }
  }

  int64_t left_row = -1, right_row = -1;
  if (seg_ok && s0 > 0) left_row = row_at<KW>(a, s0 - 1);
  if (seg_ok && s1 < a.M) right_row = row_at<KW>(a, s1);

  int64_t cur = -1;
  uint32_t curfib = 0xffffffffu;
  int run_no = 0;
  double acc[VEC], t[VEC], arow[VEC], brow[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) acc[v] = t[v] = arow[v] = brow[v] = 0.0;

  auto flush = [&](int64_t row, bool last) {
    const bool edge = ((run_no == 0) && (row == left_row)) || (last && (row == right_row));
    if (lane_active) {
      double *o = a.out + row * a.ldo + a.col0 + colv;
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        if (!colok[v]) continue;
        if (edge) red_add_f64(o + v, acc[v]);
        else o[v] = acc[v];
      }
    }
  };
  auto close_fiber = [&]() {
    if constexpr (!PHI) {
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[v] = fma(arow[v], t[v], acc[v]);
    }
  };

  int nch = (int)((s1 - s0 + G - 1) / G);
#pragma unroll
  for (int o = 16; o; o >>= 1) nch = max(nch, __shfl_xor_sync(0xffffffffu, nch, o));

  Key kn{0, 0};
  double vn = 0.0;
  if (s0 + gl < s1) {
    kn = load_key_stream<KW>(a.keys, s0 + gl);
    vn = ld_stream_f64(a.vals + s0 + gl);
  }

  const double *Fa = a.F.ptr[fm] + a.col0 + colld;
  const uint32_t lda = (uint32_t)a.F.ld[fm];
  // rest-mode bases resolved once (dynamic parameter indexing outside the loop)
  const double *fpr[NR > 0 ? NR : 1];
  uint32_t ldr[NR > 0 ? NR : 1];
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    fpr[j] = a.F.ptr[rest[j]] + a.col0 + colld;
    ldr[j] = (uint32_t)a.F.ld[rest[j]];
  }

  for (int ch = 0; ch < nch; ++ch) {
    const int64_t base = s0 + (int64_t)ch * G;
    const Key k = kn;
    const double val = vn;
    {
      const int64_t xn = base + G + gl;
      if (xn < s1) {
        kn = load_key_stream<KW>(a.keys, xn);
        vn = ld_stream_f64(a.vals + xn);
      }
    }
    uint32_t c[NM];
    uint32_t crow = 0, cfib = 0;
    uint32_t crest[NR > 0 ? NR : 1];
#pragma unroll
    for (int m = 0; m < NM; ++m) {
      c[m] = (uint32_t)decode_fast<KW>(a.L, m, k);
      if (m == mode) crow = c[m];
      if (m == fm) cfib = c[m];
    }
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      crest[j] = 0;
#pragma unroll
      for (int m = 0; m < NM; ++m)
        if (rest[j] == m) crest[j] = c[m];
    }
    const int64_t rem = s1 - base;
    const int cnt = rem <= 0 ? 0 : (rem < (int64_t)G ? (int)rem : G);
#pragma unroll
    for (int ib = 0; ib < G; ib += U) {
      int64_t row[U];
      uint32_t fib[U];
      double vv[U];
      bool ok[U], nfib[U], nrow[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        ok[u] = ib + u < cnt;
        row[u] = (int64_t)__shfl_sync(0xffffffffu, crow, gbase + ib + u);
        fib[u] = __shfl_sync(0xffffffffu, cfib, gbase + ib + u);
        vv[u] = __shfl_sync(0xffffffffu, val, gbase + ib + u);
        const int64_t prow = u ? row[u - 1] : cur;
        const uint32_t pfib = u ? fib[u - 1] : curfib;
        nrow[u] = row[u] != prow;
        nfib[u] = nrow[u] || fib[u] != pfib;
      }
      // gathers: rest-mode rows for every nonzero; the fiber row only when a
      // fiber starts; the scaled row (Phi) only when a row run starts
      double fr[NR > 0 ? NR : 1][U][VEC];
      double fa[U][VEC];
      double fb[U][VEC];
#pragma unroll
      for (int j = 0; j < NR; ++j) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t idx = __shfl_sync(0xffffffffu, crest[j], gbase + ib + u);
          load_row<VEC>(fpr[j] + (uint64_t)idx * ldr[j], true, fr[j][u]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (nfib[u] && ok[u]) load_row<VEC>(Fa + (uint64_t)fib[u] * lda, true, fa[u]);
        if constexpr (PHI) {
          if (nrow[u] && ok[u]) load_row<VEC>(a.scaled + row[u] * a.lds + a.col0 + colld, true, fb[u]);
        }
      }
      // stream-order accumulation
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if constexpr (!PHI) {
          if (ok[u]) {
            if (nfib[u]) {
              if (cur >= 0) close_fiber();
              if (nrow[u]) {
                if (cur >= 0) {
                  flush(cur, false);
                  ++run_no;
                }
                cur = row[u];
#pragma unroll
                for (int q = 0; q < VEC; ++q) acc[q] = 0.0;
              }
              curfib = fib[u];
#pragma unroll
              for (int q = 0; q < VEC; ++q) {
                arow[q] = fa[u][q];
                t[q] = 0.0;
              }
            }
            double p[VEC];
#pragma unroll
            for (int q = 0; q < VEC; ++q) p[q] = vv[u];
#pragma unroll
            for (int j = 0; j < NR; ++j)
#pragma unroll
              for (int q = 0; q < VEC; ++q) p[q] *= fr[j][u][q];
#pragma unroll
            for (int q = 0; q < VEC; ++q) t[q] += p[q];
          }
        } else {
          // Phi: krp = A_a[j] o prod_rest; d = B[i] . krp (group reduce);
          // the group reduction is warp-wide, so it runs for every slot
          if (ok[u] && nfib[u]) {
            if (nrow[u]) {
              if (cur >= 0) {
                flush(cur, false);
                ++run_no;
              }
              cur = row[u];
#pragma unroll
              for (int q = 0; q < VEC; ++q) {
                acc[q] = 0.0;
                brow[q] = fb[u][q];
              }
            }
            curfib = fib[u];
#pragma unroll
            for (int q = 0; q < VEC; ++q) arow[q] = fa[u][q];
          }
          double krp[VEC];
#pragma unroll
          for (int q = 0; q < VEC; ++q) krp[q] = arow[q];
#pragma unroll
          for (int j = 0; j < NR; ++j)
#pragma unroll
            for (int q = 0; q < VEC; ++q) krp[q] *= fr[j][u][q];
          double d = 0.0;
#pragma unroll
          for (int q = 0; q < VEC; ++q) d = fma(colok[q] ? brow[q] : 0.0, krp[q], d);
#pragma unroll
          for (int o = G / 2; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
          if (d < a.eps) d = a.eps;
          const double w = vv[u] / d;
          if (ok[u]) {
#pragma unroll
            for (int q = 0; q < VEC; ++q) acc[q] = fma(w, krp[q], acc[q]);
          }
        }
      }
    }
  }
  if (cur >= 0) {
    close_fiber();
    flush(cur, true);
  }
}

}  // namespace alto
