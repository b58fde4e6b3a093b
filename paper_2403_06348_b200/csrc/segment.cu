// ALTO line-segment MTTKRP with shared-memory output privatisation (sm_100a).
//
// The paper's conflict-resolution kernel (the reference's
// recursive strategy, pkg/src/alto/kernels.py:169-210, _jit.py:16-30,
// :53-64): one CTA per ALTO line segment [bounds[l], bounds[l+1]) streams its
// keys in ALTO order, decodes them in registers and accumulates into a
// private copy of the segment's output interval [T^s_l, T^e_l] x R held in
// shared memory; at the end the interval is added to the output with fp64
// reductions (the only global atomics: a row shared by several segments
// gets one reduction per segment, the GPU form of the pull reduction).
//
// Shared-memory fp64 atomics are CAS loops on sm_100a (ATOMS.CAST.SPIN.64),
// so the accumulation is atomic-free by construction:
//   1. a tile of T nonzeros is copied to shared memory (cp.async), every
//      thread decodes its nonzeros' coordinates and ranks them by output row
//      with an int32 shared histogram (native ATOMS.ADD);
//   2. a block scan turns the histogram into row offsets, and the decoded
//      tile is scattered into row order (SoA: rows, coordinates, values);
//   3. each group of G lanes (4 rank columns per lane) walks a contiguous
//      chunk of the row-ordered tile, gathers the other modes' factor rows
//      (256-bit loads) and sums row runs in registers. A run that lies inside
//      the chunk is added to the accumulator with a plain read-modify-write:
//      in row order no other chunk holds that row. A row that crosses chunk
//      boundaries forms a chain: the chunk where it starts owns it, the
//      others park their part in a per-chunk slot, and after a barrier the
//      owner sums the slots in chunk order and updates the accumulator once.
// The next tile's copy is in flight while a tile is processed.
#include <string.h>

#include "alto_common.cuh"
#include "run_kernels.cuh"

namespace alto {

constexpr int kSegTile = 1024;    // nonzeros per tile
// threads per CTA: 512 (one CTA per SM); 256 with two CTAs per SM is opt-in
constexpr int kSegThreadsMax = 512;
constexpr int kSegMaxBuckets = 4096;  // row-sort buckets without privatisation

struct SegArgs {
  Layout L;
  Factors F;
  const uint64_t *keys;
  const double *vals;
  int64_t M;
  const int64_t *bounds;  // [nseg + 1] balanced_bounds(M, nseg)
  const int64_t *lo;      // [nseg][N] interval lower ends (alto_partition)
  int32_t nseg;
  int32_t mode;
  int32_t rank;      // columns of this launch
  int32_t col0;      // first column of this launch
  int32_t acc_rows;  // accumulator rows (>= every segment's interval width; 0 without privatisation)
  int32_t hist_rows; // row-sort buckets (privatised: acc_rows; else rows are bucketed modulo)
  double *out;
  int64_t ldo;
};

template <int KW, int NM, int G, int NT>
struct SegLayout {
  static constexpr int RC = 4 * G;  // accumulator columns
  static constexpr int T = kSegTile;
  static constexpr int NGRP = NT / G;
  static constexpr int C = T / NGRP;  // nonzeros per group chunk
  // byte offsets after the accumulator (acc_rows * RC doubles)
  static constexpr int STAGE_KEYS = 0;
  static constexpr int STAGE_VALS = STAGE_KEYS + T * 8 * KW;
  static constexpr int SVALS = STAGE_VALS + T * 8;
  static constexpr int SROWS = SVALS + T * 8;
  static constexpr int SCRD = SROWS + T * 4;
  static constexpr int SLOT = SCRD + T * 4 * (NM - 1);  // chain slots [NGRP][RC]
  static constexpr int SLOT_ROW = SLOT + NGRP * RC * 8;
  static constexpr int HIST = SLOT_ROW + NGRP * 4;
  static constexpr int WSUM = HIST;  // the scan's warp totals follow the histogram
  static size_t bytes(int acc_rows, int hist_rows) {
    const size_t hist = ((size_t)(hist_rows + 1) * 4 + 15) & ~size_t(15);
    return (size_t)acc_rows * RC * 8 + HIST + hist + 32 * 4;
  }
};

__device__ __forceinline__ void cp_async8(void *smem, const void *gmem, int src_bytes) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async16_ca(void *smem, const void *gmem, int src_bytes) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(src_bytes) : "memory");
}

// Exclusive scan of h[0..n) in place (block of NT threads); wsum has room
// for one partial per warp.
template <int NT>
__device__ __forceinline__ void block_exclusive_scan(int32_t *h, int n, int32_t *wsum) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per = (n + NT - 1) / NT;
  const int b = tid * per;
  int32_t loc = 0;
  for (int i = 0; i < per; ++i)
    if (b + i < n) loc += h[b + i];
  int32_t inc = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int32_t w = lane < NT / 32 ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < NT / 32) wsum[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  int32_t run = inc - loc + (warp > 0 ? wsum[warp - 1] : 0);
  for (int i = 0; i < per; ++i)
    if (b + i < n) {
      const int32_t c = h[b + i];
      h[b + i] = run;
      run += c;
    }
}

template <int KW, int NM, int G, bool PRIV, int NT>
__global__ void __launch_bounds__(NT, kSegThreadsMax / NT) alto_segment_kernel(const __grid_constant__ SegArgs a) {
  using SL = SegLayout<KW, NM, G, NT>;
  constexpr int T = SL::T, C = SL::C, RC = SL::RC, VEC = kVec;
  constexpr int NO = NM - 1;
  constexpr int U = NO >= 3 ? 2 : 4;  // nonzeros per gather batch (divides C; measured: U = 2 for 4+ modes)
  constexpr int PER = T / NT;  // tile nonzeros per thread in the sort
  constexpr uint32_t kNone = 0xffffffffu;
  extern __shared__ __align__(16) unsigned char seg_smem[];
  double *acc = reinterpret_cast<double *>(seg_smem);
  unsigned char *base = seg_smem + (PRIV ? (size_t)a.acc_rows * RC * 8 : 0);
  unsigned char *stage_keys = base + SL::STAGE_KEYS;
  double *stage_vals = reinterpret_cast<double *>(base + SL::STAGE_VALS);
  double *svals = reinterpret_cast<double *>(base + SL::SVALS);
  uint32_t *srows = reinterpret_cast<uint32_t *>(base + SL::SROWS);
  uint32_t *scrd = reinterpret_cast<uint32_t *>(base + SL::SCRD);
  double *slot = reinterpret_cast<double *>(base + SL::SLOT);
  uint32_t *slot_row = reinterpret_cast<uint32_t *>(base + SL::SLOT_ROW);
  int32_t *hist = reinterpret_cast<int32_t *>(base + SL::HIST);
  const int hist_n = a.hist_rows;
  int32_t *wsum = hist + ((hist_n + 1 + 3) & ~3);

  const int tid = threadIdx.x;
  const int g = tid / G, gl = tid & (G - 1);
  const int seg = blockIdx.x;
  const int64_t s0 = a.bounds[seg], s1 = a.bounds[seg + 1];
  const int64_t lo = a.lo[(int64_t)seg * a.L.nmodes + a.mode];
  const int mode = a.mode;

  const int colv = gl * VEC;
  bool colok[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) colok[v] = colv + v < a.rank;
  const bool lane_active = colok[0];
  const int colld = lane_active ? colv : 0;
  const char *fb[NO];
  uint32_t fldb[NO];
#pragma unroll
  for (int j = 0; j < NO; ++j) {
    const int mj = j < mode ? j : j + 1;
    fb[j] = reinterpret_cast<const char *>(a.F.ptr[mj] + a.col0 + colld);
    fldb[j] = (uint32_t)(a.F.ld[mj] * 8);
  }

  if constexpr (PRIV) {
    for (int i = tid; i < a.acc_rows * RC; i += NT) acc[i] = 0.0;
  }
  for (int i = tid; i < hist_n; i += NT) hist[i] = 0;

  auto issue = [&](int64_t t0) {
    const int64_t n = s1 - t0 < T ? s1 - t0 : T;
    for (int i = tid; i < T; i += NT) {
      const bool in = i < n;
      const int64_t x = in ? t0 + i : 0;
      if constexpr (KW == 1) cp_async8(stage_keys + i * 8, a.keys + x, in ? 8 : 0);
      else cp_async16_ca(stage_keys + i * 16, a.keys + 2 * x, in ? 16 : 0);
      cp_async8(stage_vals + i, a.vals + x, in ? 8 : 0);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  if (s0 < s1) issue(s0);
  for (int64_t t0 = s0; t0 < s1; t0 += T) {
    const int cnt = (int)(s1 - t0 < T ? s1 - t0 : T);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();  // tile staged; previous tile's accumulation done; histogram zeroed
    // 1. decode + rank by output row
    uint32_t crd[PER][NM];
    uint32_t lrow[PER];
    int32_t rk[PER];
    double vl[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int p = tid + k * NT;
      rk[k] = -1;
      if (p < cnt) {
        Key key;
        if constexpr (KW == 1) {
          key.w0 = reinterpret_cast<const uint64_t *>(stage_keys)[p];
          key.w1 = 0;
        } else {
          const ulonglong2 kk = reinterpret_cast<const ulonglong2 *>(stage_keys)[p];
          key.w0 = kk.x;
          key.w1 = kk.y;
        }
        uint32_t r = 0;
#pragma unroll
        for (int m = 0; m < NM; ++m) {
          crd[k][m] = (uint32_t)decode_fast<KW>(a.L, m, key);
          if (m == mode) r = crd[k][m];
        }
        vl[k] = stage_vals[p];
        lrow[k] = r - (uint32_t)lo;
        rk[k] = atomicAdd(&hist[PRIV ? lrow[k] : lrow[k] % (uint32_t)hist_n], 1);
      }
    }
    __syncthreads();
    // 2. row offsets, scatter into row order
    block_exclusive_scan<NT>(hist, hist_n, wsum);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      if (rk[k] >= 0) {
        const uint32_t lr = lrow[k];
        const int pos = hist[PRIV ? lr : lr % (uint32_t)hist_n] + rk[k];
        srows[pos] = lr;
        svals[pos] = vl[k];
#pragma unroll
        for (int j = 0; j < NO; ++j) scrd[j * T + pos] = j < mode ? crd[k][j] : crd[k][j + 1];
      }
    }
    __syncthreads();  // row-ordered tile complete; stage and histogram free
    if (t0 + T < s1) issue(t0 + T);
    for (int i = tid; i < hist_n; i += NT) hist[i] = 0;

    // 3. group chunks of the row-ordered tile
    const int p0 = g * C;
    const int p1 = p0 + C < cnt ? p0 + C : cnt;
    const uint32_t left_row = (p0 > 0 && p0 < cnt) ? srows[p0 - 1] : kNone;
    const uint32_t right_row = p1 < cnt ? srows[p1] : kNone;
    uint32_t cur = kNone;
    bool first = true;
    double run[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) run[v] = 0.0;

    auto flush = [&](uint32_t r, bool is_first, bool is_last) {
      if constexpr (!PRIV) {
        if (lane_active) {
          double *o = a.out + ((int64_t)lo + r) * a.ldo + a.col0 + colv;
#pragma unroll
          for (int v = 0; v < VEC; ++v)
            if (colok[v]) red_add_f64(o + v, run[v]);
        }
        return;
      } else {
        const bool from_left = is_first && r == left_row;
        const bool to_right = is_last && r == right_row;
        if (from_left) {
          // part of a chain started in an earlier chunk: park it
          double *s = slot + g * RC + colv;
#pragma unroll
          for (int v = 0; v < VEC; ++v) s[v] = run[v];
          if (gl == 0) slot_row[g] = r;
        } else if (!to_right) {
          double *o = acc + (int64_t)r * RC + colv;
#pragma unroll
          for (int v = 0; v < VEC; ++v) o[v] += run[v];
        }
        // to_right && !from_left: chain head, kept in registers (below)
      }
    };

    if (p0 < cnt) {
      for (int q = p0; q < p1; q += U) {
        uint32_t row[U];
        double vv[U];
        double f[NO][U][VEC];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const bool in = q + u < p1;
          row[u] = in ? srows[q + u] : kNone;
          vv[u] = in ? svals[q + u] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < NO; ++j)
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const uint32_t idx = q + u < p1 ? scrd[j * T + q + u] : 0u;
            load_row<VEC>(reinterpret_cast<const double *>(fb[j] + (uint64_t)idx * fldb[j]), true, f[j][u]);
          }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (row[u] == kNone) continue;
          if (row[u] != cur) {
            if (cur != kNone) {
              flush(cur, first, false);
              first = false;
            }
            cur = row[u];
#pragma unroll
            for (int v = 0; v < VEC; ++v) run[v] = 0.0;
          }
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            double t = vv[u] * f[0][u][v];
#pragma unroll
            for (int j = 1; j < NO; ++j) t *= f[j][u][v];
            run[v] += t;
          }
        }
      }
      if (cur != kNone) flush(cur, first, true);
    }
    if constexpr (PRIV) {
      __syncthreads();  // parked chain parts visible
      // chain heads: the chunk where a row crossing chunk boundaries starts
      // adds the parts of the following chunks in chunk order
      const bool head = p0 < cnt && cur != kNone && cur == right_row && !(first && cur == left_row);
      if (head) {
        int h = g + 1;
        while (true) {
          const double *s = slot + h * RC + colv;
#pragma unroll
          for (int v = 0; v < VEC; ++v) run[v] += s[v];
          const int e = (h + 1) * C;
          if (e < cnt && srows[e] == cur) ++h;
          else break;
        }
        double *o = acc + (int64_t)cur * RC + colv;
#pragma unroll
        for (int v = 0; v < VEC; ++v) o[v] += run[v];
      }
    }
  }
  if constexpr (PRIV) {
    __syncthreads();
    // the segment's interval -> output (one reduction per touched entry)
    const int n = a.acc_rows * RC;
    for (int i = tid; i < n; i += NT) {
      const int r = i / RC, c = i - r * RC;
      const double v = acc[i];
      if (c < a.rank && v != 0.0) red_add_f64(a.out + ((int64_t)lo + r) * a.ldo + a.col0 + c, v);
    }
  }
}

size_t segment_smem_bytes(int words, int nmodes, int g, int nt, int64_t acc_rows, int64_t hist_rows) {
  // SegLayout's constants, spelled out for the host
  const size_t fixed = (size_t)kSegTile * (8 * words + 8 + 8 + 4 + 4 * (nmodes - 1)) +
                       (size_t)(nt / g) * (4 * g * 8 + 4);
  const size_t hist = ((size_t)(hist_rows + 1) * 4 + 15) & ~size_t(15);
  return (size_t)acc_rows * 4 * g * 8 + fixed + hist + 32 * 4;
}

template <int KW, int NM, int G, bool PRIV, int NT>
static int launch_seg(const SegArgs &a, cudaStream_t st) {
  using SL = SegLayout<KW, NM, G, NT>;
  const size_t smem = SL::bytes(PRIV ? a.acc_rows : 0, a.hist_rows);
  auto k = alto_segment_kernel<KW, NM, G, PRIV, NT>;
  ALTO_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k<<<a.nseg, NT, smem, st>>>(a);
  ALTO_LAUNCH_CHECK("alto_segment_kernel");
  return ALTO_OK;
}

template <int KW, int NM, bool PRIV, int NT>
static int dispatch_g(const SegArgs &a, int g, cudaStream_t st) {
  switch (g) {
    case 2: return launch_seg<KW, NM, 2, PRIV, NT>(a, st);
    case 4: return launch_seg<KW, NM, 4, PRIV, NT>(a, st);
    default: return launch_seg<KW, NM, 8, PRIV, NT>(a, st);
  }
}

template <int KW, bool PRIV, int NT>
static int dispatch_nm(const SegArgs &a, int g, cudaStream_t st) {
  switch (a.L.nmodes) {
    case 3: return dispatch_g<KW, 3, PRIV, NT>(a, g, st);
    case 4: return dispatch_g<KW, 4, PRIV, NT>(a, g, st);
    default: return dispatch_g<KW, 5, PRIV, NT>(a, g, st);
  }
}

// Launch shape: G lanes per nonzero (4 * G accumulator columns: the rank in
// column chunks) and NT threads. The widest G whose accumulator fits, then
// 256 threads if two CTAs fit on an SM.
struct SegShape {
  int g, nt;
  size_t smem;
};

static SegShape seg_shape(int words, int nmodes, int rank, int64_t acc_rows, int64_t hist_rows, bool priv,
                          size_t optin, size_t per_sm) {
  int g = 2;
  while (g < 8 && 4 * g < rank) g *= 2;
  const int64_t acc = priv ? acc_rows : 0;
  while (g > 2 && segment_smem_bytes(words, nmodes, g, kSegThreadsMax, acc, hist_rows) > optin) g /= 2;
  SegShape s{g, kSegThreadsMax, segment_smem_bytes(words, nmodes, g, kSegThreadsMax, acc, hist_rows)};
  // two 256-thread CTAs per SM measured slower than one of 512 (c3 mode 3:
  // 15.8 vs 11.1-12.6 ms): opt-in only
  const size_t s256 = segment_smem_bytes(words, nmodes, g, 256, acc, hist_rows);
  if (2 * (s256 + 1024) <= per_sm && getenv("ALTO_B200_SEG_NT256")) s = SegShape{g, 256, s256};
  return s;
}

static int launch_segment(const SegArgs &base, int words, bool priv, const SegShape &sh, cudaStream_t st) {
  const int R = base.F.rank;
  const int rc = 4 * sh.g;
  for (int c0 = 0; c0 < R; c0 += rc) {
    SegArgs a = base;
    a.col0 = c0;
    a.rank = R - c0 < rc ? R - c0 : rc;
    int r;
    if (sh.nt == 256) {
      if (words == 1) r = priv ? dispatch_nm<1, true, 256>(a, sh.g, st) : dispatch_nm<1, false, 256>(a, sh.g, st);
      else r = priv ? dispatch_nm<2, true, 256>(a, sh.g, st) : dispatch_nm<2, false, 256>(a, sh.g, st);
    } else {
      if (words == 1) r = priv ? dispatch_nm<1, true, 512>(a, sh.g, st) : dispatch_nm<1, false, 512>(a, sh.g, st);
      else r = priv ? dispatch_nm<2, true, 512>(a, sh.g, st) : dispatch_nm<2, false, 512>(a, sh.g, st);
    }
    if (r) return r;
  }
  return ALTO_OK;
}

static int device_smem(size_t *optin, size_t *per_sm) {
  int dev = 0, a = 0, b = 0;
  ALTO_CUDA(cudaGetDevice(&dev));
  ALTO_CUDA(cudaDeviceGetAttribute(&a, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  ALTO_CUDA(cudaDeviceGetAttribute(&b, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
  *optin = (size_t)a;
  *per_sm = (size_t)b;
  return ALTO_OK;
}

}  // namespace alto

using namespace alto;

extern "C" {

int alto_segment_smem_bytes(int32_t word_bits, int32_t nmodes, int32_t rank, int64_t acc_rows,
                            size_t *host_bytes) {
  ALTO_REQUIRE(host_bytes != nullptr, ALTO_ERR_VALUE, "null output");
  ALTO_REQUIRE(nmodes >= 3 && nmodes <= 5, ALTO_ERR_UNSUPPORTED, "segment kernel: 3..5 modes");
  size_t optin = 0, per_sm = 0;
  int rc = device_smem(&optin, &per_sm);
  if (rc) {  // no device (build container): assume B200's limits
    optin = 232448;
    per_sm = 233472;
  }
  *host_bytes = seg_shape(word_bits == 128 ? 2 : 1, nmodes, rank, acc_rows, acc_rows, true, optin, per_sm).smem;
  return ALTO_OK;
}

int alto_mttkrp_segment(const alto_layout_t *host_layout, const void *keys, const double *vals, int64_t M,
                        const alto_factors_t *host_factors, int32_t mode, double *out, int64_t ldo,
                        const int64_t *bounds, const int64_t *lo, int32_t L, int64_t acc_rows,
                        int32_t privatize, void *stream) {
  int rc = check_layout(host_layout);
  if (rc) return rc;
  rc = check_factors(host_layout, host_factors);
  if (rc) return rc;
  ALTO_REQUIRE(mode >= 0 && mode < host_layout->nmodes, ALTO_ERR_VALUE, "mode %d out of range", mode);
  ALTO_REQUIRE(host_layout->nmodes >= 3 && host_layout->nmodes <= 5, ALTO_ERR_UNSUPPORTED,
               "segment kernel: 3..5 modes");
  if (M == 0) return ALTO_OK;
  ALTO_REQUIRE(L >= 1 && bounds != nullptr && lo != nullptr, ALTO_ERR_VALUE, "need segment tables");
  for (int n = 0; n < host_layout->nmodes; ++n)
    ALTO_REQUIRE(host_layout->dims[n] <= 0xfffffffeLL, ALTO_ERR_UNSUPPORTED, "segment kernel: dims < 2^32");
  ALTO_REQUIRE(acc_rows >= 1, ALTO_ERR_VALUE, "acc_rows must be >= 1");
  const int words = host_layout->word_bits == 128 ? 2 : 1;
  // without privatisation acc_rows only sizes the row-sort histogram
  const int64_t hist_rows = privatize ? acc_rows : (acc_rows < kSegMaxBuckets ? acc_rows : kSegMaxBuckets);
  size_t optin = 0, per_sm = 0;
  rc = device_smem(&optin, &per_sm);
  if (rc) return rc;
  const SegShape sh = seg_shape(words, host_layout->nmodes, host_factors->rank, acc_rows, hist_rows,
                                privatize != 0, optin, per_sm);
  ALTO_REQUIRE(sh.smem <= optin, ALTO_ERR_UNSUPPORTED,
               "segment interval of %lld rows needs %zu B of shared memory (> %zu)", (long long)acc_rows, sh.smem,
               optin);
  SegArgs a;
  memset(&a, 0, sizeof a);
  a.L = to_device_layout(host_layout);
  a.F = to_device_factors(host_factors);
  a.keys = static_cast<const uint64_t *>(keys);
  a.vals = vals;
  a.M = M;
  a.bounds = bounds;
  a.lo = lo;
  a.nseg = L;
  a.mode = mode;
  a.acc_rows = privatize ? (int32_t)acc_rows : 0;
  a.hist_rows = (int32_t)hist_rows;
  a.out = out;
  a.ldo = ldo;
  return launch_segment(a, words, privatize != 0, sh, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
