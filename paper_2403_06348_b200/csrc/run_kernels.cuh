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
#ifndef RUN_U
#define RUN_U 4
#endif
#ifndef RUN_VEC
#define RUN_VEC 4
#endif
constexpr int kVec = RUN_VEC;  // doubles per lane per factor row (4: 32-byte sectors)

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
  if constexpr (VEC == 4) {
    // 256-bit gather (LDG.E.ENL2.256 on sm_100a): one 32-byte sector per lane
    if (ok) {
#if defined(GATHER_CG)
      asm volatile("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];"
                   : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3])
                   : "l"(p));
#elif defined(GATHER_EL)
      asm volatile("ld.global.nc.L1::evict_last.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
                   : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3])
                   : "l"(p), "l"(l2_policy_evict_last()));
#elif defined(GATHER_L2EL)
      asm volatile("ld.global.nc.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
                   : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3])
                   : "l"(p), "l"(l2_policy_evict_last()));
#elif defined(GATHER_NOALLOC)
      asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];"
                   : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3])
                   : "l"(p));
#else
      asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                   : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3])
                   : "l"(p));
#endif
    } else {
      r[0] = r[1] = r[2] = r[3] = 0.0;
    }
  } else if constexpr (VEC == 2) {
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
  return (int64_t)decode_fast<KW>(a.L, a.mode, load_key<KW>(a.keys, x));
}

// Gathered contribution of one nonzero, before accumulation.
template <int VEC>
struct Contribution {
  int64_t row;
  double p[VEC];  // MTTKRP: v * prod rows; Phi: krp
  double w;       // Phi: v / max(d, eps)
};

template <int NM, int G, int VEC, int KW, bool PHI, bool EXACT, bool ATOMIC>
__global__ void __launch_bounds__(256, 2) run_kernel(const __grid_constant__ RunArgs a) {
  constexpr int U = G < RUN_U ? G : RUN_U;  // nonzeros gathered per batch (loads in flight)
  // Control flow is warp-uniform so every shuffle runs with the full mask;
  // groups whose segment is shorter (or absent) just carry predicates.
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int gbase = lane & ~(G - 1);  // first lane of this group
  const int64_t seg = gtid / G;
  const bool seg_ok = seg < a.nseg;
  const int64_t s0 = seg_ok ? seg_begin(seg, a.M, a.nseg) : a.M;
  const int64_t s1 = seg_ok ? seg_begin(seg + 1, a.M, a.nseg) : a.M;
  const int N = NM > 0 ? NM : a.L.nmodes;
  const int mode = a.mode;

  const int colv = gl * VEC;  // first column (within chunk) of this lane
  bool colok[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) colok[v] = colv + v < a.rank;
  const bool lane_active = colok[0];
  const int colld = lane_active ? colv : 0;  // idle lanes gather column 0

  int64_t left_row = -1, right_row = -1;
  if constexpr (!ATOMIC) {
    if (seg_ok && s0 > 0) left_row = row_at<KW>(a, s0 - 1);
    if (seg_ok && s1 < a.M) right_row = row_at<KW>(a, s1);
  }

  int64_t cur = -1;
  int run_no = 0;
  double acc[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) acc[v] = 0.0;

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
      const int slot = from_left ? 0 : (to_right ? 1 : -1);
      if (slot < 0) {
        if (lane_active) {
          double *o = a.out + row * a.ldo + a.col0 + colv;
#pragma unroll
          for (int v = 0; v < VEC; ++v)
            if (colok[v]) o[v] = acc[v];
        }
      } else if constexpr (!EXACT) {
        // fast path: a run cut by a segment edge is reduced straight into
        // the (zeroed) output; a hot row split over thousands of segments
        // costs one fp64 reduction per segment instead of a serial merge
        if (lane_active) {
          double *o = a.out + row * a.ldo + a.col0 + colv;
#pragma unroll
          for (int v = 0; v < VEC; ++v)
            if (colok[v]) red_add_f64(o + v, acc[v]);
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

  // warp-uniform chunk count
  int nch = (int)((s1 - s0 + G - 1) / G);
#pragma unroll
  for (int o = 16; o; o >>= 1) nch = max(nch, __shfl_xor_sync(0xffffffffu, nch, o));

  // software pipeline: the next chunk's (key, value) is in flight while the
  // current chunk is gathered
  Key kn{0, 0};
  double vn = 0.0;
  if (s0 + gl < s1) {
    kn = load_key_stream<KW>(a.keys, s0 + gl);
    vn = ld_stream_f64(a.vals + s0 + gl);
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
    // in-register decode (coordinates < 2^32 on the fast path)
    uint32_t c[NM > 0 ? NM : 1];
    uint32_t crow;
    if constexpr (NM > 0) {
      crow = 0;
#pragma unroll
      for (int m = 0; m < NM; ++m) {
#ifdef ABL_NO_DECODE
        c[m] = (uint32_t)((k.w0 >> (m * 7)) % (uint64_t)a.L.dims[m]);
#else
        c[m] = (uint32_t)decode_fast<KW>(a.L, m, k);
#endif
        if (m == mode) crow = c[m];
      }
    } else {
      crow = (uint32_t)decode_fast<KW>(a.L, mode, k);
    }
    const int64_t rem = s1 - base;
    const int cnt = rem <= 0 ? 0 : (rem < (int64_t)G ? (int)rem : G);
#pragma unroll
    for (int ib = 0; ib < G; ib += U) {
      Contribution<VEC> cb[U];
      bool ok[U];
      double vv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        ok[u] = ib + u < cnt;
        cb[u].row = (int64_t)__shfl_sync(0xffffffffu, crow, gbase + ib + u);
        vv[u] = __shfl_sync(0xffffffffu, val, gbase + ib + u);
#pragma unroll
        for (int q = 0; q < VEC; ++q) cb[u].p[q] = PHI ? 1.0 : vv[u];
      }
      // Gathers are unconditional (indices of idle slots decode to valid
      // rows, idle lanes read column 0) so all loads of the batch issue
      // back to back before the first use.
      if (PHI && a.pi != nullptr) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t xs = ok[u] ? base + ib + u : 0;
          load_row<VEC>(a.pi + xs * a.ldp + a.col0 + colld, true, cb[u].p);
        }
      } else if constexpr (NM > 0) {
        // the NM-1 other modes in ascending order; mode j of the list is
        // j or j+1 (no per-mode branches, so every load stays in flight)
        double f[NM - 1][U][VEC];
#pragma unroll
        for (int j = 0; j < NM - 1; ++j) {
          const int mj = j < mode ? j : j + 1;
          const uint32_t cj = j < mode ? c[j] : c[j + 1];
          const double *fm = a.F.ptr[mj] + a.col0 + colld;
          const uint32_t ldm = (uint32_t)a.F.ld[mj];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const uint32_t idx = __shfl_sync(0xffffffffu, cj, gbase + ib + u);
#ifdef ABL_NO_GATHER
            for (int q = 0; q < VEC; ++q) f[j][u][q] = 1.0 + (double)(idx & 1);
#else
            load_row<VEC>(fm + (uint64_t)idx * ldm, true, f[j][u]);
#endif
          }
        }
#pragma unroll
        for (int j = 0; j < NM - 1; ++j)
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int q = 0; q < VEC; ++q) cb[u].p[q] = mul<EXACT>(cb[u].p[q], f[j][u][q]);
      } else {
        // generic mode count: decode the broadcast key per nonzero
#pragma unroll
        for (int u = 0; u < U; ++u) {
          Key kb;
          kb.w0 = __shfl_sync(0xffffffffu, k.w0, gbase + ib + u);
          kb.w1 = KW == 2 ? __shfl_sync(0xffffffffu, k.w1, gbase + ib + u) : 0ull;
          for (int m = 0; m < N; ++m) {
            if (m == mode) continue;
            const uint64_t idx = decode_fast<KW>(a.L, m, kb);
            double f[VEC];
            load_row<VEC>(a.F.ptr[m] + (int64_t)idx * a.F.ld[m] + a.col0 + colld, true, f);
#pragma unroll
            for (int q = 0; q < VEC; ++q) cb[u].p[q] = mul<EXACT>(cb[u].p[q], f[q]);
          }
        }
      }
      if constexpr (PHI) {
        double brow[U][VEC];
#pragma unroll
        for (int u = 0; u < U; ++u)
          load_row<VEC>(a.scaled + cb[u].row * a.lds + a.col0 + colld, true, brow[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          double d = 0.0;
          if constexpr (EXACT) {
            // sequential over r as the reference does (pkg/src/alto/_jit.py:94-96)
            double t[VEC];
#pragma unroll
            for (int q = 0; q < VEC; ++q) t[q] = colok[q] ? __dmul_rn(brow[u][q], cb[u].p[q]) : 0.0;
#pragma unroll
            for (int j = 0; j < G; ++j) {
#pragma unroll
              for (int q = 0; q < VEC; ++q) {
                const double tj = __shfl_sync(0xffffffffu, t[q], gbase + j);
                if (j * VEC + q < a.rank) d = __dadd_rn(d, tj);
              }
            }
          } else {
#pragma unroll
            for (int q = 0; q < VEC; ++q) d = fma(colok[q] ? brow[u][q] : 0.0, cb[u].p[q], d);
#pragma unroll
            for (int o = G / 2; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
          }
          if (d < a.eps) d = a.eps;
          cb[u].w = __ddiv_rn(vv[u], d);
        }
      }
      // accumulate in stream order: row runs stay in registers
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (ok[u]) {
          if (cb[u].row != cur) {
            if (cur >= 0) {
              flush(cur, false);
              ++run_no;
            }
            cur = cb[u].row;
#pragma unroll
            for (int q = 0; q < VEC; ++q) acc[q] = 0.0;
          }
#pragma unroll
          for (int q = 0; q < VEC; ++q)
            acc[q] = PHI ? add<EXACT>(acc[q], mul<EXACT>(cb[u].w, cb[u].p[q])) : add<EXACT>(acc[q], cb[u].p[q]);
        }
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
