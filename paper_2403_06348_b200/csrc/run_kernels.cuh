// Templated MTTKRP / Phi stream kernels (sm_100a).
//
// One kernel body serves two traversals of a nonzero stream:
//   * ATOMIC = false: a mode-ordered view (rows contiguous). Every lane group
//     owns one balanced segment, accumulates each row run in registers in
//     stream order and writes it once; runs that cross a segment edge go to a
//     per-segment edge buffer that merge_edges_kernel folds in ascending
//     segment order. This is the reference's output-oriented strategy
//     (pkg/src/alto/kernels.py:213-252, pkg/src/alto/_jit.py:33-50) and is
//     bit-identical to it for the same segment count.
//   * ATOMIC = true: the ALTO-ordered stream itself; row runs are flushed with
//     fp64 reductions (red.global.add.f64) -- the direct-atomic strategy of the
//     paper's adaptive conflict resolution.
//
// Work mapping: a group of G lanes handles one nonzero at a time, each lane
// owning VEC consecutive rank columns (rank-vectorised 16-byte gathers). The
// group first loads G consecutive (key, value) pairs coalesced, each lane
// decodes its own key (in-register bit extraction), then the group walks the
// G nonzeros broadcasting coordinates with width-G shuffles.
#pragma once

#include "alto_common.cuh"

namespace alto {

constexpr int kMaxRankChunk = 32;

struct RunArgs {
  Layout L;
  Factors F;
  const uint64_t *keys;
  const double *vals;
  int64_t M;
  int32_t mode;
  int32_t rank;  // columns handled by this launch (<= 32)
  int32_t col0;  // first column of this launch
  int32_t full_rank;
  int64_t nseg;
  double *out;
  int64_t ldo;
  // edge buffers (ATOMIC = false)
  int64_t *edge_row;     // [2 * nseg]: first-run row / last-run row, -1 when direct
  int32_t *edge_through; // [nseg]
  double *edge_val;      // [2 * nseg][kMaxRankChunk]
  // Phi
  const double *scaled;
  int64_t lds;
  const double *pi;
  int64_t ldp;
  double eps;
};

template <int G>
__device__ __forceinline__ unsigned group_mask() {
  if constexpr (G == 32) return 0xffffffffu;
  const unsigned lane = threadIdx.x & 31;
  return ((1u << G) - 1u) << (lane & ~(G - 1));
}

template <int G, typename T>
__device__ __forceinline__ T gshfl(unsigned mask, T v, int src) {
  return __shfl_sync(mask, v, src, G);
}

template <int VEC>
__device__ __forceinline__ void load_row(const double *p, bool ok, double (&r)[VEC]) {
  if constexpr (VEC == 2) {
    if (ok) {
      const double2 t = __ldg(reinterpret_cast<const double2 *>(p));
      r[0] = t.x;
      r[1] = t.y;
    } else {
      r[0] = r[1] = 0.0;
    }
  } else {
    r[0] = ok ? __ldg(p) : 0.0;
  }
}

template <bool EXACT>
__device__ __forceinline__ double mul(double a, double b) {
  if constexpr (EXACT) return __dmul_rn(a, b);
  else return a * b;
}
template <bool EXACT>
__device__ __forceinline__ double add(double a, double b) {
  if constexpr (EXACT) return __dadd_rn(a, b);
  else return a + b;
}

__device__ __forceinline__ int64_t seg_begin(int64_t s, int64_t M, int64_t L) {
  const int64_t base = M / L, extra = M % L;
  return s * base + (s < extra ? s : extra);
}

template <int KW>
__device__ __forceinline__ int64_t row_at(const RunArgs &a, int64_t x) {
  return (int64_t)decode_mode(a.L, a.mode, load_key<KW>(a.keys, x));
}

template <int NM, int G, int VEC, int KW, bool PHI, bool EXACT, bool ATOMIC>
__global__ void __launch_bounds__(256) run_kernel(const __grid_constant__ RunArgs a) {
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int gl = threadIdx.x & (G - 1);
  const int64_t seg = gtid / G;
  if (seg >= a.nseg) return;  // whole groups exit together
  const unsigned gm = group_mask<G>();
  const int64_t s0 = seg_begin(seg, a.M, a.nseg);
  const int64_t s1 = seg_begin(seg + 1, a.M, a.nseg);
  const int N = NM > 0 ? NM : a.L.nmodes;
  const int mode = a.mode;

  const int colv = gl * VEC;  // first column (within chunk) of this lane
  bool colok[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) colok[v] = colv + v < a.rank;
  const bool lane_active = colok[0];

  int64_t left_row = -1, right_row = -1;
  if constexpr (!ATOMIC) {
    if (s0 > 0) left_row = row_at<KW>(a, s0 - 1);
    if (s1 < a.M) right_row = row_at<KW>(a, s1);
  }

  int64_t cur = -1;
  int run_no = 0;
  double acc[VEC];
  double brow[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) acc[v] = brow[v] = 0.0;

  auto flush = [&](int64_t row, bool last) {
    if constexpr (ATOMIC) {
      if (lane_active) {
        double *o = a.out + row * a.ldo + a.col0 + colv;
#pragma unroll
        for (int v = 0; v < VEC; ++v)
          if (colok[v]) red_add_f64(o + v, acc[v]);
      }
    } else {
      const bool from_left = (run_no == 0) && (row == left_row);
      const bool to_right = last && (row == right_row);
      int slot = -1;
      if (from_left) slot = 0;
      else if (to_right) slot = 1;
      if (slot < 0) {
        if (lane_active) {
          double *o = a.out + row * a.ldo + a.col0 + colv;
#pragma unroll
          for (int v = 0; v < VEC; ++v)
            if (colok[v]) o[v] = acc[v];
        }
      } else {
        double *e = a.edge_val + (2 * seg + slot) * kMaxRankChunk + colv;
        if (lane_active) {
#pragma unroll
          for (int v = 0; v < VEC; ++v)
            if (colok[v]) e[v] = acc[v];
        }
        if (gl == 0) {
          a.edge_row[2 * seg + slot] = row;
          if (slot == 0 && to_right) a.edge_through[seg] = 1;
        }
      }
    }
  };

  for (int64_t base = s0; base < s1; base += G) {
    const int64_t x = base + gl;
    const bool valid = x < s1;
    Key k{0, 0};
    double val = 0.0;
    if (valid) {
      k = load_key_stream<KW>(a.keys, x);
      val = ld_stream_f64(a.vals + x);
    }
    uint64_t c[NM > 0 ? NM : 1];
    uint64_t crow = 0;
    if constexpr (NM > 0) {
#pragma unroll
      for (int m = 0; m < NM; ++m) {
        c[m] = decode_mode(a.L, m, k);
        if (m == mode) crow = c[m];
      }
    } else {
      crow = decode_mode(a.L, mode, k);
    }
    const int cnt = (int)(s1 - base < (int64_t)G ? s1 - base : (int64_t)G);
    for (int it = 0; it < cnt; ++it) {
      const int64_t row = (int64_t)gshfl<G>(gm, crow, it);
      const double v = gshfl<G>(gm, val, it);
      if (row != cur) {
        if (cur >= 0) {
          flush(cur, false);
          ++run_no;
        }
        cur = row;
#pragma unroll
        for (int q = 0; q < VEC; ++q) acc[q] = 0.0;
        if constexpr (PHI) {
          double t[VEC];
          load_row<VEC>(a.scaled + row * a.lds + a.col0 + colv, lane_active, t);
#pragma unroll
          for (int q = 0; q < VEC; ++q) brow[q] = colok[q] ? t[q] : 0.0;
        }
      }
      // product of the other modes' factor rows, ascending mode order
      double p[VEC];
#pragma unroll
      for (int q = 0; q < VEC; ++q) p[q] = PHI ? 1.0 : v;
      if (PHI && a.pi != nullptr) {
        const int64_t xs = base + it;
        load_row<VEC>(a.pi + xs * a.ldp + a.col0 + colv, lane_active, p);
      } else {
        Key kb;
        if constexpr (NM == 0) {
          kb.w0 = gshfl<G>(gm, k.w0, it);
          kb.w1 = KW == 2 ? gshfl<G>(gm, k.w1, it) : 0ull;
        }
#pragma unroll
        for (int m = 0; m < (NM > 0 ? NM : ALTO_MAX_MODES); ++m) {
          if (NM == 0 && m >= N) break;
          if (m == mode) continue;
          uint64_t idx;
          if constexpr (NM > 0) idx = gshfl<G>(gm, c[m], it);
          else idx = decode_mode(a.L, m, kb);
          double f[VEC];
          load_row<VEC>(a.F.ptr[m] + (int64_t)idx * a.F.ld[m] + a.col0 + colv, lane_active, f);
#pragma unroll
          for (int q = 0; q < VEC; ++q) p[q] = mul<EXACT>(p[q], f[q]);
        }
      }
      if constexpr (PHI) {
        // d = sum_r scaled[row, r] * krp[r]
        double d = 0.0;
        if constexpr (EXACT) {
          // sequential over r as the reference does (pkg/src/alto/_jit.py:94-96)
          double t[VEC];
#pragma unroll
          for (int q = 0; q < VEC; ++q) t[q] = colok[q] ? __dmul_rn(brow[q], p[q]) : 0.0;
          const int nl = (a.rank + VEC - 1) / VEC;
          for (int j = 0; j < nl; ++j) {
#pragma unroll
            for (int q = 0; q < VEC; ++q) {
              const double tj = gshfl<G>(gm, t[q], j);
              if (j * VEC + q < a.rank) d = __dadd_rn(d, tj);
            }
          }
        } else {
#pragma unroll
          for (int q = 0; q < VEC; ++q) d = fma(brow[q], colok[q] ? p[q] : 0.0, d);
#pragma unroll
          for (int o = G / 2; o; o >>= 1) d += __shfl_xor_sync(gm, d, o, G);
        }
        if (d < a.eps) d = a.eps;
        const double w = __ddiv_rn(v, d);
#pragma unroll
        for (int q = 0; q < VEC; ++q) acc[q] = add<EXACT>(acc[q], mul<EXACT>(w, p[q]));
      } else {
#pragma unroll
        for (int q = 0; q < VEC; ++q) acc[q] = add<EXACT>(acc[q], p[q]);
      }
    }
  }
  if (cur >= 0) flush(cur, true);
}

// host-side dispatch (instantiations live in run_kw{1,2}_{mttkrp,phi}.cu)
int launch_run(const RunArgs &a, int words, bool phi, bool exact, bool atomic, cudaStream_t st);
int launch_run_kw1_mttkrp(const RunArgs &a, int nm, int g, bool exact, bool atomic, int grid, cudaStream_t st);
int launch_run_kw2_mttkrp(const RunArgs &a, int nm, int g, bool exact, bool atomic, int grid, cudaStream_t st);
int launch_run_kw1_phi(const RunArgs &a, int nm, int g, bool exact, bool atomic, int grid, cudaStream_t st);
int launch_run_kw2_phi(const RunArgs &a, int nm, int g, bool exact, bool atomic, int grid, cudaStream_t st);

}  // namespace alto
