// Memoised CP-ALS sweep for 3-mode tensors, consumer side and the piece
// index (see memo0_kernel in dview_kernels.cu for the producer).
//
// CP-ALS updates the modes in order (pkg/src/alto/cpd/als.py:84-96); with
// modes (m0, m1, k) the MTTKRPs of m0 and m1 share the partial sums over
// the third mode's rows, which do not change between the two updates:
//   T[i, j] = sum_k v_ijk A_k[k]
//   MTTKRP_m0[i] = sum_j A_m1[j] o T[i, j]      (memo0_kernel)
//   MTTKRP_m1[j] = sum_i A_m0'[i] o T[i, j]     (memo1_kernel, below)
// T is kept per "piece" (a run of equal (i, j) inside one 512-nonzero
// segment of m0's view; a fiber cut by a segment edge is two pieces, which
// the sum above does not mind), stored in piece order by the producer;
// memo1 walks the pieces sorted by (j, i) through a position -> piece index
// (pid), reading one 8R-byte T row and gathering one factor row per piece
// instead of two factor rows per nonzero. Summation order differs from the
// reference's (fast path; <= 1e-12 relative in the tests).
#include "alto_common.cuh"
#include "det.cuh"
#include "run_kernels.cuh"

namespace alto {
namespace {

constexpr int kSegM = 512;  // segment of m0's decoded view (dview_kernels.cu kDvSeg)

// pieces per segment: a piece starts at the segment's first nonzero and
// wherever (row, j) changes. One warp per segment, 32 consecutive nonzeros
// per step (coalesced), starts counted with a ballot.
__device__ __forceinline__ uint32_t piece_starts(const uint32_t *__restrict__ rows, const uint32_t *__restrict__ jc,
                                                 int64_t x, int64_t s0, int64_t s1, bool *start) {
  const bool in = x < s1;
  const uint32_t r = in ? rows[x] : 0u, j = in ? jc[x] : 0u;
  const bool first = x == s0;
  const uint32_t pr = (in && !first) ? rows[x - 1] : 0u, pj = (in && !first) ? jc[x - 1] : 0u;
  *start = in && (first || r != pr || j != pj);
  return __ballot_sync(0xffffffffu, *start);
}

__global__ void memo_count_kernel(const uint32_t *__restrict__ rows, const uint32_t *__restrict__ jc, int64_t M,
                                  int64_t nseg, uint32_t *__restrict__ counts) {
  const int lane = threadIdx.x & 31;
  for (int64_t seg = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; seg < nseg;
       seg += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t s0 = seg * kSegM, s1 = s0 + kSegM < M ? s0 + kSegM : M;
    uint32_t n = 0;
    for (int64_t b = s0; b < s1; b += 32) {
      bool st;
      n += __popc(piece_starts(rows, jc, b + lane, s0, s1, &st));
    }
    if (lane == 0) counts[seg] = n;
  }
}

// exclusive scan of n counts into out[0..n] (out[n] = total), one block
__global__ void memo_scan_kernel(const uint32_t *__restrict__ counts, int64_t n, uint32_t *__restrict__ out) {
  __shared__ uint64_t part[1024];
  const int t = threadIdx.x, T = blockDim.x;
  const int64_t per = (n + T - 1) / T;
  const int64_t b = t * per, e = b + per < n ? b + per : n;
  uint64_t s = 0;
  for (int64_t i = b; i < e; ++i) s += counts[i];
  part[t] = s;
  __syncthreads();
  if (t == 0) {
    uint64_t acc = 0;
    for (int i = 0; i < T; ++i) {
      const uint64_t v = part[i];
      part[i] = acc;
      acc += v;
    }
    out[n] = (uint32_t)acc;
  }
  __syncthreads();
  uint64_t acc = part[t];
  for (int64_t i = b; i < e; ++i) {
    out[i] = (uint32_t)acc;
    acc += counts[i];
  }
}

__global__ void memo_emit_kernel(const uint32_t *__restrict__ rows, const uint32_t *__restrict__ jc, int64_t M,
                                 int64_t nseg, const uint32_t *__restrict__ pbase, uint64_t nrows,
                                 uint64_t *__restrict__ keys, uint64_t *__restrict__ ids) {
  const int lane = threadIdx.x & 31;
  const uint32_t below = (1u << lane) - 1u;
  for (int64_t seg = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; seg < nseg;
       seg += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t s0 = seg * kSegM, s1 = s0 + kSegM < M ? s0 + kSegM : M;
    uint32_t p = pbase[seg];
    for (int64_t b = s0; b < s1; b += 32) {
      bool st;
      const uint32_t m = piece_starts(rows, jc, b + lane, s0, s1, &st);
      if (st) {
        const uint32_t q = p + __popc(m & below);
        keys[q] = (uint64_t)jc[b + lane] * nrows + rows[b + lane];  // consumer order: (j, i)
        ids[q] = q;
      }
      p += __popc(m);
    }
  }
}

__global__ void memo_finish_kernel(const uint64_t *__restrict__ keys, const uint64_t *__restrict__ ids, int64_t P,
                                   uint64_t nrows, uint32_t *__restrict__ prow, uint32_t *__restrict__ pcrd,
                                   uint32_t *__restrict__ pid) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < P; x += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[x];
    prow[x] = (uint32_t)(k / nrows);
    pcrd[x] = (uint32_t)(k % nrows);
    pid[x] = (uint32_t)ids[x];
  }
}

// blocks of 256 threads for one warp per segment (grid-stride past 16 per SM)
int seg_warp_blocks(int64_t nseg) {
  int64_t b = (nseg + 7) / 8;
  const int64_t cap = (int64_t)num_sms() * 16;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

struct Memo1Args {
  const uint32_t *prow;  // [P] output row (j) of every piece, ascending
  const uint32_t *pcrd;  // [P] row of the gathered factor (i)
  const uint32_t *pid;   // [P] piece (row of T) at every position; null: position == piece
  const double *T;       // [P][ldT], piece order
  int64_t ldT;
  int64_t P;
  const double *A;  // gathered factor (mode m0, updated)
  int64_t lda;
  double *out;
  int64_t ldo;
  int32_t rank;
  int32_t col0;
  DetEdges det;  // deterministic mode (det.cu), or det.val == null
};

__device__ __forceinline__ void ld_stream4(const double *p, bool ok, double (&r)[4]) {
  if (ok) {
    // T rows are read once: evict-first in L2 keeps the gathered factor rows
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
                 : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3])
                 : "l"(p), "l"(l2_policy_evict_first()));
  } else {
    r[0] = r[1] = r[2] = r[3] = 0.0;
  }
}

// group of G lanes per 512-piece segment, 4 columns per lane; batches of 4
// pieces: 4 factor-row gathers + 4 streamed T rows in flight, the next
// batch's (row, i) prefetched
template <int G, bool DET>
__global__ void __launch_bounds__(256) memo1_kernel(const __grid_constant__ Memo1Args a) {
  constexpr int VEC = kVec, U = 4;
  static_assert(U == 4, "load4 reads uint4");
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, gl = lane & (G - 1);
  const int64_t seg = gtid / G;
  const int64_t s0 = seg * kSegM < a.P ? seg * kSegM : a.P;
  const int64_t s1 = s0 + kSegM < a.P ? s0 + kSegM : a.P;
  const bool seg_ok = s0 < s1;
  const int colv = gl * VEC;
  bool colok[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) colok[v] = colv + v < a.rank;
  const bool lane_active = colok[0];
  const int colld = lane_active ? colv : 0;
  constexpr uint32_t kNone = 0xffffffffu;
  const uint32_t left_row = (seg_ok && s0 > 0) ? a.prow[s0 - 1] : kNone;
  const uint32_t right_row = (seg_ok && s1 < a.P) ? a.prow[s1] : kNone;
  const double *Ab = a.A + a.col0 + colld;
  const double *Tb = a.T + a.col0 + colld;

  uint32_t cur = kNone;
  int run_no = 0;
  double acc[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) acc[v] = 0.0;
  auto flush = [&](uint32_t row, bool last) {
    const bool from_left = (run_no == 0) && (row == left_row), to_right = last && (row == right_row);
    const bool edge = from_left || to_right;
    if constexpr (DET) {
      if (edge) {
        det_park<VEC>(a.det, seg, from_left, to_right, row, acc, colv, gl, lane_active);
        return;
      }
    }
    if (lane_active) {
      double *o = a.out + (int64_t)row * a.ldo + a.col0 + colv;
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        if (!colok[v]) continue;
        if (edge) red_add_f64(o + v, acc[v]);
        else o[v] = acc[v];
      }
    }
  };
  // the group's 4 pieces of a batch: one 128-bit load per array (x is a
  // multiple of 4: segments start at multiples of 512), scalar at the tail
  auto load4 = [&](int64_t x, uint32_t (&r)[U], uint32_t (&c)[U], uint32_t (&id)[U]) {
    if (x + U <= s1) {
      const uint4 r4 = __ldg(reinterpret_cast<const uint4 *>(a.prow + x));
      const uint4 c4 = __ldg(reinterpret_cast<const uint4 *>(a.pcrd + x));
      r[0] = r4.x, r[1] = r4.y, r[2] = r4.z, r[3] = r4.w;
      c[0] = c4.x, c[1] = c4.y, c[2] = c4.z, c[3] = c4.w;
      if (a.pid != nullptr) {
        const uint4 i4 = __ldg(reinterpret_cast<const uint4 *>(a.pid + x));
        id[0] = i4.x, id[1] = i4.y, id[2] = i4.z, id[3] = i4.w;
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) id[u] = (uint32_t)(x + u);  // pieces in T order
      }
      return;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool in = x + u < s1;
      r[u] = in ? __ldg(a.prow + x + u) : kNone;
      c[u] = in ? __ldg(a.pcrd + x + u) : 0u;
      id[u] = in ? (a.pid != nullptr ? __ldg(a.pid + x + u) : (uint32_t)(x + u)) : 0u;
    }
  };

  int nb = (int)((s1 - s0 + U - 1) / U);
#pragma unroll
  for (int o = 16; o; o >>= 1) nb = max(nb, __shfl_xor_sync(0xffffffffu, nb, o));
  uint32_t rn[U], cn[U], in_[U];
  load4(s0, rn, cn, in_);
  for (int b = 0; b < nb; ++b) {
    const int64_t x = s0 + (int64_t)b * U;
    uint32_t r[U], c[U], id[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      r[u] = rn[u];
      c[u] = cn[u];
      id[u] = in_[u];
    }
    if (b + 1 < nb) load4(x + U, rn, cn, in_);
    double fa[U][VEC], ft[U][VEC];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ok = x + u < s1;
      load_row<VEC>(Ab + (int64_t)c[u] * a.lda, ok, fa[u]);
      ld_stream4(Tb + (int64_t)id[u] * a.ldT, ok, ft[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (x + u < s1) {
        if (r[u] != cur) {
          if (cur != kNone) {
            flush(cur, false);
            ++run_no;
          }
          cur = r[u];
#pragma unroll
          for (int q = 0; q < VEC; ++q) acc[q] = 0.0;
        }
#pragma unroll
        for (int q = 0; q < VEC; ++q) acc[q] = fma(fa[u][q], ft[u][q], acc[q]);
      }
    }
  }
  // all 32/G groups of the warp ending in one row (a hot row spanning the
  // warp's segments): sum their runs with a fixed shuffle tree and reduce
  // once, instead of 32/G fp64 reductions of the same addresses
  const uint32_t r0 = __shfl_sync(0xffffffffu, cur, 0);
  if (G < 32 && !DET && __all_sync(0xffffffffu, cur == r0 && cur != kNone)) {
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      double x = acc[v];
#pragma unroll
      for (int k = 16; k >= G; k >>= 1) x += __shfl_xor_sync(0xffffffffu, x, k);
      acc[v] = x;
    }
    if (lane < G && lane_active) {
      double *o = a.out + (int64_t)cur * a.ldo + a.col0 + colv;
#pragma unroll
      for (int v = 0; v < VEC; ++v)
        if (colok[v]) red_add_f64(o + v, acc[v]);
    }
  } else if (cur != kNone) {
    flush(cur, true);
  }
}

}  // namespace
}  // namespace alto

using namespace alto;

extern "C" {

int alto_memo_pieces_count(const uint32_t *rows, const uint32_t *jcrd, int64_t M, uint32_t *counts,
                           uint32_t *pbase, void *stream) {
  ALTO_REQUIRE(M > 0, ALTO_ERR_VALUE, "empty tensor");
  const int64_t nseg = (M + kSegM - 1) / kSegM;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  memo_count_kernel<<<seg_warp_blocks(nseg), 256, 0, st>>>(rows, jcrd, M, nseg, counts);
  ALTO_LAUNCH_CHECK("memo_count_kernel");
  memo_scan_kernel<<<1, 1024, 0, st>>>(counts, nseg, pbase);
  ALTO_LAUNCH_CHECK("memo_scan_kernel");
  return ALTO_OK;
}

int alto_memo_sort_scratch_bytes(int64_t P, size_t *host_bytes) {
  *host_bytes = radix_sort_scratch(P < 1 ? 1 : P, 1);
  return ALTO_OK;
}

int alto_memo_pieces_build(const uint32_t *rows, const uint32_t *jcrd, int64_t M, const uint32_t *pbase,
                           int64_t P, int64_t nrows_m0, int64_t nrows_m1, uint64_t *keys, uint64_t *ids,
                           void *scratch, size_t scratch_bytes, uint32_t *prow, uint32_t *pcrd, uint32_t *pid,
                           void *stream) {
  ALTO_REQUIRE(M > 0 && P > 0 && P < (int64_t)0xffffffffll, ALTO_ERR_VALUE, "bad piece count");
  const int64_t nseg = (M + kSegM - 1) / kSegM;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  memo_emit_kernel<<<seg_warp_blocks(nseg), 256, 0, st>>>(rows, jcrd, M, nseg, pbase, (uint64_t)nrows_m0,
                                                               keys, ids);
  ALTO_LAUNCH_CHECK("memo_emit_kernel");
  int bits = 1;
  while (bits < 64 && ((uint64_t)1 << bits) < (uint64_t)nrows_m0 * (uint64_t)nrows_m1) ++bits;
  int rc = radix_sort_pairs(1, bits, keys, ids, P, scratch, scratch_bytes, st);
  if (rc) return rc;
  int64_t blocks = (P + 255) / 256;
  if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
  memo_finish_kernel<<<(int)blocks, 256, 0, st>>>(keys, ids, P, (uint64_t)nrows_m0, prow, pcrd, pid);
  ALTO_LAUNCH_CHECK("memo_finish_kernel");
  return ALTO_OK;
}

int alto_mttkrp_memo1(const uint32_t *prow, const uint32_t *pcrd, const uint32_t *pid, const double *T,
                      int64_t ldT, int64_t P,
                      const double *A, int64_t lda, int32_t rank, double *out, int64_t ldo, void *stream) {
  ALTO_REQUIRE(rank >= 1, ALTO_ERR_VALUE, "rank must be positive");
  if (P <= 0) return ALTO_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Memo1Args a;
  a.prow = prow;
  a.pcrd = pcrd;
  a.pid = pid;
  a.T = T;
  a.ldT = ldT;
  a.P = P;
  a.A = A;
  a.lda = lda;
  a.out = out;
  a.ldo = ldo;
  a.det = DetEdges{nullptr, nullptr, nullptr};
  for (int c0 = 0; c0 < rank; c0 += kMaxRankChunk) {
    a.col0 = c0;
    a.rank = rank - c0 < kMaxRankChunk ? rank - c0 : kMaxRankChunk;
    int g = 1;
    while (g * kVec < a.rank) g *= 2;
    const int grid = (int)ceil_div(ceil_div(P, kSegM) * g, 256);
    const int64_t nseg = ceil_div(P, kSegM);
    if (det_enabled()) {
      const int rc = det_edges(nseg, &a.det, st);
      if (rc) return rc;
    }
    const bool det = a.det.val != nullptr;
#define MEMO1(GV)                                            \
  if (det) memo1_kernel<GV, true><<<grid, 256, 0, st>>>(a);  \
  else memo1_kernel<GV, false><<<grid, 256, 0, st>>>(a);
    switch (g) {
      case 1: MEMO1(1) break;
      case 2: MEMO1(2) break;
      case 4: MEMO1(4) break;
      default: MEMO1(8) break;
    }
#undef MEMO1
    ALTO_LAUNCH_CHECK("memo1_kernel");
    if (a.det.val != nullptr) {
      const int rc = det_merge(a.det, nseg, a.out, a.ldo, a.col0, a.rank, st);
      if (rc) return rc;
    }
  }
  return ALTO_OK;
}


}  // extern "C"
