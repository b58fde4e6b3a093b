// Piece sums of the memoised CP-ALS sweep, branch-free (split producer).
//
// The producing mode m0 of a memoised pair (memo.py) needs, per piece p = a
// run of equal (i, j) inside one 512-nonzero segment of m0's fiber view,
//   T[p] = sum_{x in p} v_x A_k[k_x]
// (the reference recomputes every MTTKRP, pkg/src/alto/cpd/als.py:84-96; this
// is the shared dimension-tree term of modes m0 and m1). Pieces average 5-7
// nonzeros on c2, so the row-run machinery of dview3 (a divergent flush
// branch per run end) ran ~54 warp instructions per nonzero step. Here a
// piece start is one bit of the stream and the kernel has no data-dependent
// branch: per nonzero one 256-bit gather of A_k[k], v * A_k[k] accumulated in
// registers, and a predicated 256-bit streaming store of the closed piece
// (pieces of a segment are consecutive T rows from pbase[seg], so the store
// address advances by one row per piece start).
//
// Stream (interleaved layout of dview.cuh, built by alto_memo_sums_stream):
//   kf[x] = k_x | (x starts a piece) << 31      u32
//   v[x]                                         f64
// 12 B per nonzero, staged per warp with bulk copies; zero padding extends
// the last piece with zeros.
#include "dview.cuh"

namespace alto {

namespace {

struct SumsArgs {
  const uint32_t *kf;
  const double *vals;
  int64_t M;
  int64_t Mp;  // interleaved length
  const double *Ak;
  int64_t ldk;
  int32_t rank;
  const uint32_t *pbase;  // [nseg + 1] first piece of every segment
  double *T;
  int64_t ldT;
};

#ifndef SUMS_MINB
#define SUMS_MINB 4
#endif
#ifndef SUMS_STAGES
#define SUMS_STAGES 3
#endif
constexpr int kSumsStages = SUMS_STAGES;
constexpr int kSumsHead = 128;
constexpr int kSumsStage = kIlWarpChunk * 4 + kIlWarpChunk * 8;
constexpr int kSumsWarp = kSumsHead + kSumsStage * kSumsStages;

template <int G>
__global__ void __launch_bounds__(256, SUMS_MINB) memo_sums_kernel(const __grid_constant__ SumsArgs a) {
  extern __shared__ __align__(16) unsigned char sm_smem[];
  constexpr int VEC = kVec, NG = 32 / G, CH = 4 * G, Q = G, S = kSumsStages;
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int grp = lane / G;
  const int64_t seg = gtid / G;
  const int64_t s0 = seg * kDvSeg < a.M ? seg * kDvSeg : a.M;
  const int64_t s1 = s0 + kDvSeg < a.M ? s0 + kDvSeg : a.M;
  unsigned char *wbase = sm_smem + (threadIdx.x >> 5) * kSumsWarp;
  uint64_t *bars = reinterpret_cast<uint64_t *>(wbase);
  const int64_t wblk = gtid >> 5;

  const int colv = gl * VEC;
  const bool lane_active = colv < a.rank;
  const int colld = lane_active ? colv : 0;
  const char *fb = reinterpret_cast<const char *>(a.Ak + colld);
  const uint32_t ldkb = (uint32_t)(a.ldk * 8);

  // T row of the open piece: the first piece start advances to pbase[seg]
  const bool seg_ok = s0 < s1;
  double *tp = a.T + ((int64_t)(seg_ok ? a.pbase[seg] : 0u) - 1) * a.ldT + colv;
  const int64_t tstep = a.ldT;
  bool open = false;
  double acc[VEC];
#pragma unroll
  for (int q = 0; q < VEC; ++q) acc[q] = 0.0;

  auto issue = [&](int c, int slot) {
    if (lane == 0) {
      unsigned char *st = wbase + kSumsHead + slot * kSumsStage;
      const int64_t src = wblk * (NG * kDvSeg) + (int64_t)c * kIlWarpChunk;
      fence_proxy_async();
      mbar_expect_tx(&bars[slot], kSumsStage);
      bulk_g2s(st, a.kf + src, kIlWarpChunk * 4, &bars[slot]);
      bulk_g2s(st + kIlWarpChunk * 4, a.vals + src, kIlWarpChunk * 8, &bars[slot]);
    }
  };

  int nch = (int)((s1 - s0 + CH - 1) / CH);
#pragma unroll
  for (int o = 16; o; o >>= 1) nch = max(nch, __shfl_xor_sync(0xffffffffu, nch, o));
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    fence_proxy_async();
  }
  __syncwarp();
#pragma unroll
  for (int c = 0; c < S - 1; ++c)
    if (c < nch) issue(c, c);

  const bool store_ok = lane_active;
  for (int ch = 0; ch < nch; ++ch) {
    __syncwarp();
    if (ch + S - 1 < nch) issue(ch + S - 1, (ch + S - 1) % S);
    mbar_wait(&bars[ch % S], (uint32_t)((ch / S) & 1));
    const unsigned char *st = wbase + kSumsHead + (ch % S) * kSumsStage;
    // quad k of this group: piece-start flags + k coordinates, values
    auto quad = [&](int k, uint32_t (&kf)[4], double (&vv)[4]) {
      const uint4 kf4 = *reinterpret_cast<const uint4 *>(st + k * 16 * NG + grp * 16);
      const unsigned char *sv = st + kIlWarpChunk * 4 + k * 32 * NG + grp * 16;
      const double2 v01 = *reinterpret_cast<const double2 *>(sv);
      const double2 v23 = *reinterpret_cast<const double2 *>(sv + 16 * NG);
      kf[0] = kf4.x, kf[1] = kf4.y, kf[2] = kf4.z, kf[3] = kf4.w;
      vv[0] = v01.x, vv[1] = v01.y, vv[2] = v23.x, vv[3] = v23.y;
    };
    auto gather = [&](const uint32_t (&kf)[4], double (&f)[4][VEC]) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        load_row<VEC>(reinterpret_cast<const double *>(fb + (uint64_t)(kf[u] & 0x7fffffffu) * ldkb), true, f[u]);
    };
    auto consume = [&](const uint32_t (&kf)[4], const double (&vv)[4], const double (&f)[4][VEC]) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool np = (kf[u] >> 31) != 0;
        st_cs_v4_if(tp, np && open && store_ok, acc);
        tp += np ? tstep : 0;
        open = open || np;
        const double keep = np ? 0.0 : 1.0;
#pragma unroll
        for (int q = 0; q < VEC; ++q) acc[q] = fma(acc[q], keep, vv[u] * f[u][q]);
      }
    };
#pragma unroll 1
    for (int k = 0; k < Q; ++k) {
      uint32_t kf[4];
      double vv[4], f[4][VEC];
      quad(k, kf, vv);
      gather(kf, f);
      consume(kf, vv, f);
    }
  }
  st_cs_v4_if(tp, open && store_ok, acc);
}

// ---- fused producer: piece sums + this mode's MTTKRP, branch-free ---------
//
// The producing mode's own MTTKRP, out_m0[i] = sum_x A_m1[j_x] o (v_x A_k[k_x]),
// is accumulated from the same products (A_m1's row gathered once per piece
// with a predicated load issued with the batch's A_k gathers, held while the
// piece lasts), so T is written once and never read back by the producer. Stream (interleaved): rows (u32),
// jf = j | piece-start << 31 (u32), k (u32), v (f64) = 20 B per nonzero.
// Output rows: runs privatised in registers, written once, fp64 reductions
// for runs cut by a segment edge (dview3's scheme; the flush branch is taken
// once per row run, rows average thousands of nonzeros).
// cache hints of the fused kernel's gathers (A/B knobs): A_j rows are read
// once per piece in ascending j inside a row run
#ifndef FUSED_JHINT
#define FUSED_JHINT 1  // 0: default, 1: L1::no_allocate, 2: L1::evict_first
#endif
#ifndef FUSED_KHINT
#define FUSED_KHINT 0  // 0: default, 1: L1::evict_last
#endif
__device__ __forceinline__ void fused_load_j(const double *p, bool pred, double (&r)[4]) {
#if FUSED_JHINT == 1
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t@q ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];\n\t}"
      : "+d"(r[0]), "+d"(r[1]), "+d"(r[2]), "+d"(r[3])
      : "l"(p), "r"((int)pred));
#elif FUSED_JHINT == 2
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t@q ld.global.nc.L1::evict_first.v4.f64 {%0, %1, %2, %3}, [%4];\n\t}"
      : "+d"(r[0]), "+d"(r[1]), "+d"(r[2]), "+d"(r[3])
      : "l"(p), "r"((int)pred));
#else
  load_row_if(p, pred, r);
#endif
}
__device__ __forceinline__ void fused_load_k(const double *p, double (&r)[4]) {
#if FUSED_KHINT == 1
  asm volatile("ld.global.nc.L1::evict_last.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3])
               : "l"(p));
#else
  load_row<4>(p, true, r);
#endif
}
#ifndef FUSED_U
#define FUSED_U 2
#endif
#ifndef FUSED_MINB
#define FUSED_MINB 2
#endif
#ifndef FUSED_STAGES
#define FUSED_STAGES 2
#endif
constexpr int kFusedStages = FUSED_STAGES;
constexpr int kFusedStage = kIlWarpChunk * 4 * 3 + kIlWarpChunk * 8;
constexpr int kFusedWarp = kSumsHead + kFusedStage * kFusedStages;

struct FusedArgs {
  const uint32_t *rows;  // interleaved
  const uint32_t *jf;
  const uint32_t *kc;
  const double *vals;
  int64_t M;
  int64_t Mp;
  const double *Aj;  // next mode m1's factor (one row per piece)
  int64_t ldj;
  const double *Ak;  // third mode's factor (one row per nonzero)
  int64_t ldk;
  int32_t rank;
  const uint32_t *pbase;
  double *T;  // null: plain fiber-factored MTTKRP (no piece sums stored)
  int64_t ldT;
  double *out;
  int64_t ldo;
};

template <int G>
__global__ void __launch_bounds__(256, FUSED_MINB) memo_fused_kernel(const __grid_constant__ FusedArgs a) {
  extern __shared__ __align__(16) unsigned char fu_smem[];
  constexpr int VEC = kVec, NG = 32 / G, CH = 4 * G, Q = G, S = kFusedStages, U = FUSED_U;
  constexpr uint32_t kNone = 0xffffffffu;
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int grp = lane / G;
  const int64_t seg = gtid / G;
  const int64_t s0 = seg * kDvSeg < a.M ? seg * kDvSeg : a.M;
  const int64_t s1 = s0 + kDvSeg < a.M ? s0 + kDvSeg : a.M;
  unsigned char *wbase = fu_smem + (threadIdx.x >> 5) * kFusedWarp;
  uint64_t *bars = reinterpret_cast<uint64_t *>(wbase);
  const int64_t wblk = gtid >> 5;

  const int colv = gl * VEC;
  bool colok[VEC];
#pragma unroll
  for (int q = 0; q < VEC; ++q) colok[q] = colv + q < a.rank;
  const bool lane_active = colok[0];
  const int colld = lane_active ? colv : 0;
  const char *fk = reinterpret_cast<const char *>(a.Ak + colld);
  const char *fj = reinterpret_cast<const char *>(a.Aj + colld);
  const uint32_t ldkb = (uint32_t)(a.ldk * 8), ldjb = (uint32_t)(a.ldj * 8);

  const bool seg_ok = s0 < s1;
  const bool store_t = a.T != nullptr;
  double *tp = store_t ? a.T + ((int64_t)(seg_ok ? a.pbase[seg] : 0u) - 1) * a.ldT + colv : nullptr;
  const int64_t tstep = store_t ? a.ldT : 0;
  const uint32_t left_row = (seg_ok && s0 > 0) ? a.rows[il_u32<G>(s0 - 1)] : kNone;
  const uint32_t right_row = (seg_ok && s1 < a.M) ? a.rows[il_u32<G>(s1)] : kNone;

  uint32_t cur = kNone;
  int run_no = 0;
  bool open = false;
  double acc[VEC], tq[VEC], jcur[VEC];
#pragma unroll
  for (int q = 0; q < VEC; ++q) acc[q] = tq[q] = jcur[q] = 0.0;

  auto flush = [&](uint32_t row, bool last) {
    const bool edge = ((run_no == 0) && (row == left_row)) || (last && (row == right_row));
    if (!lane_active) return;
    double *o = a.out + (int64_t)row * a.ldo + colv;
    if (!edge && colok[VEC - 1] && (a.ldo & 3) == 0) {
      asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(o), "d"(acc[0]), "d"(acc[1]), "d"(acc[2]),
                   "d"(acc[3])
                   : "memory");
      return;
    }
#pragma unroll
    for (int q = 0; q < VEC; ++q) {
      if (!colok[q]) continue;
      if (edge) red_add_f64(o + q, acc[q]);
      else o[q] = acc[q];
    }
  };

  auto issue = [&](int c, int slot) {
    if (lane == 0) {
      unsigned char *st = wbase + kSumsHead + slot * kFusedStage;
      const int64_t src = wblk * (NG * kDvSeg) + (int64_t)c * kIlWarpChunk;
      constexpr int U32B = kIlWarpChunk * 4;
      fence_proxy_async();
      mbar_expect_tx(&bars[slot], kFusedStage);
      bulk_g2s(st, a.rows + src, U32B, &bars[slot]);
      bulk_g2s(st + U32B, a.jf + src, U32B, &bars[slot]);
      bulk_g2s(st + 2 * U32B, a.kc + src, U32B, &bars[slot]);
      bulk_g2s(st + 3 * U32B, a.vals + src, kIlWarpChunk * 8, &bars[slot]);
    }
  };

  int nch = (int)((s1 - s0 + CH - 1) / CH);
#pragma unroll
  for (int o = 16; o; o >>= 1) nch = max(nch, __shfl_xor_sync(0xffffffffu, nch, o));
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    fence_proxy_async();
  }
  __syncwarp();
#pragma unroll
  for (int c = 0; c < S - 1; ++c)
    if (c < nch) issue(c, c);

  for (int ch = 0; ch < nch; ++ch) {
    __syncwarp();
    if (ch + S - 1 < nch) issue(ch + S - 1, (ch + S - 1) % S);
    mbar_wait(&bars[ch % S], (uint32_t)((ch / S) & 1));
    const unsigned char *st = wbase + kSumsHead + (ch % S) * kFusedStage;
#pragma unroll 1
    for (int k = 0; k < Q; ++k) {
#pragma unroll
      for (int ub = 0; ub < 4; ub += U) {
        // this batch's U nonzeros of quad k (half a quad per 64-bit shared
        // read when U = 2: the quad is not held in registers)
        constexpr int U32B = kIlWarpChunk * 4;
        static_assert(U == 2 || U == 4, "batches of 2 or 4 nonzeros");
        const int off = k * 16 * NG + grp * 16 + (U == 2 ? ub * 4 : 0);
        uint32_t rr[U], jv[U], kv[U];
        double vv[U];
        if constexpr (U == 2) {
          const uint2 r2 = *reinterpret_cast<const uint2 *>(st + off);
          const uint2 j2 = *reinterpret_cast<const uint2 *>(st + U32B + off);
          const uint2 k2 = *reinterpret_cast<const uint2 *>(st + 2 * U32B + off);
          const double2 v2 = *reinterpret_cast<const double2 *>(st + 3 * U32B + k * 32 * NG + grp * 16 + ub * 8 * NG);
          rr[0] = r2.x, rr[1] = r2.y, jv[0] = j2.x, jv[1] = j2.y, kv[0] = k2.x, kv[1] = k2.y;
          vv[0] = v2.x, vv[1] = v2.y;
        } else {
          const uint4 r4 = *reinterpret_cast<const uint4 *>(st + off);
          const uint4 j4 = *reinterpret_cast<const uint4 *>(st + U32B + off);
          const uint4 k4 = *reinterpret_cast<const uint4 *>(st + 2 * U32B + off);
          const unsigned char *sv = st + 3 * U32B + k * 32 * NG + grp * 16;
          const double2 v01 = *reinterpret_cast<const double2 *>(sv);
          const double2 v23 = *reinterpret_cast<const double2 *>(sv + 16 * NG);
          rr[0] = r4.x, rr[1] = r4.y, rr[2] = r4.z, rr[3] = r4.w;
          jv[0] = j4.x, jv[1] = j4.y, jv[2] = j4.z, jv[3] = j4.w;
          kv[0] = k4.x, kv[1] = k4.y, kv[2] = k4.z, kv[3] = k4.w;
          vv[0] = v01.x, vv[1] = v01.y, vv[2] = v23.x, vv[3] = v23.y;
        }
        double f[U][VEC], g[U][VEC];
#pragma unroll
        for (int u = 0; u < U; ++u) fused_load_k(reinterpret_cast<const double *>(fk + (uint64_t)kv[u] * ldkb), f[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t jx = jv[u];
          fused_load_j(reinterpret_cast<const double *>(fj + (uint64_t)(jx & 0x7fffffffu) * ldjb), (jx >> 31) != 0,
                       g[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          // padding past the last nonzero is zeros without a piece-start
          // bit: it extends the open piece by exact zeros
          const bool np = (jv[u] >> 31) != 0;
          const bool nr = np && rr[u] != cur;
          // the closed piece's T row (predicated streaming store)
          st_cs_v4_if(tp, np && open && store_t && lane_active, tq);
          // a finished row run is flushed (rare: rows hold thousands of
          // nonzeros); the branch only reads acc and the run restarts through
          // the multiplier, so the common path moves no registers
          if (nr && cur != kNone) {
            flush(cur, false);
            ++run_no;
          }
          cur = nr ? rr[u] : cur;
          if (np) tp += tstep;
          open = open || np;
          const double kp = np ? 0.0 : 1.0, kr = nr ? 0.0 : 1.0;
#pragma unroll
          for (int q = 0; q < VEC; ++q) {
            jcur[q] = np ? g[u][q] : jcur[q];
            const double x = vv[u] * f[u][q];  // v A_k[k]
            tq[q] = fma(tq[q], kp, x);
            acc[q] = fma(acc[q], kr, jcur[q] * x);  // out_i += A_j[j] o (v A_k[k])
          }
        }
      }
    }
  }
  st_cs_v4_if(tp, open && store_t && lane_active, tq);
  // every group of the warp ending in one row: one shuffle-tree sum, one
  // reduction (a hot row spanning the warp's segments)
  if constexpr (G < 32) {
    const uint32_t r0 = __shfl_sync(0xffffffffu, cur, 0);
    if (__all_sync(0xffffffffu, cur == r0 && cur != kNone)) {
#pragma unroll
      for (int q = 0; q < VEC; ++q) {
        double x = acc[q];
#pragma unroll
        for (int o = 16; o >= G; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        acc[q] = x;
      }
      if (lane < G && lane_active) {
        double *o = a.out + (int64_t)cur * a.ldo + colv;
#pragma unroll
        for (int q = 0; q < VEC; ++q)
          if (colok[q]) red_add_f64(o + q, acc[q]);
      }
      return;
    }
  }
  if (cur != kNone) flush(cur, true);
}

template <int G>
__global__ void fused_stream_kernel(const uint32_t *__restrict__ rows, const uint32_t *__restrict__ jcrd,
                                    const uint32_t *__restrict__ kcrd, const double *__restrict__ vals, int64_t M,
                                    int64_t Mp, uint32_t *__restrict__ orows, uint32_t *__restrict__ ojf,
                                    uint32_t *__restrict__ okc, double *__restrict__ ovals) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < Mp; x += (int64_t)gridDim.x * blockDim.x) {
    uint32_t r = 0u, jf = 0u, kc = 0u;
    double v = 0.0;
    if (x < M) {
      r = rows[x];
      const uint32_t j = jcrd[x];
      const bool start = (x % kDvSeg) == 0 || r != rows[x - 1] || j != jcrd[x - 1];
      jf = j | (start ? 0x80000000u : 0u);
      kc = kcrd[x];
      v = vals[x];
    }
    const int64_t pu = il_u32<G>(x);
    orows[pu] = r;
    ojf[pu] = jf;
    okc[pu] = kc;
    ovals[il_f64<G>(x)] = v;
  }
}

// (k | piece-start bit, value) of m0's fiber view in the interleaved layout
template <int G>
__global__ void sums_stream_kernel(const uint32_t *__restrict__ rows, const uint32_t *__restrict__ jcrd,
                                   const uint32_t *__restrict__ kcrd, const double *__restrict__ vals, int64_t M,
                                   int64_t Mp, uint32_t *__restrict__ okf, double *__restrict__ ovals) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < Mp; x += (int64_t)gridDim.x * blockDim.x) {
    uint32_t kf = 0u;
    double v = 0.0;
    if (x < M) {
      const bool start = (x % kDvSeg) == 0 || rows[x] != rows[x - 1] || jcrd[x] != jcrd[x - 1];
      kf = kcrd[x] | (start ? 0x80000000u : 0u);
      v = vals[x];
    }
    okf[il_u32<G>(x)] = kf;
    ovals[il_f64<G>(x)] = v;
  }
}

int sums_group(int rank) {
  int g = 1;
  while (g * kVec < rank) g *= 2;
  return g;
}

}  // namespace

}  // namespace alto

using namespace alto;

extern "C" {

int alto_memo_sums_stream(const uint32_t *rows, const uint32_t *jcrd, const uint32_t *kcrd, const double *vals,
                          int64_t M, int32_t rank, uint32_t *il_kf, double *il_vals, void *stream) {
  ALTO_REQUIRE(M >= 0, ALTO_ERR_VALUE, "negative nnz");
  ALTO_REQUIRE(rank >= 1 && rank <= kMaxRankChunk, ALTO_ERR_UNSUPPORTED, "piece sums support rank <= %d",
               kMaxRankChunk);
  const int g = sums_group(rank);
  const int64_t Mp = il_len(M < 1 ? 1 : M, g);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t blocks = ceil_div(Mp, 256);
  if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
#define SSK(GV) sums_stream_kernel<GV><<<(int)blocks, 256, 0, st>>>(rows, jcrd, kcrd, vals, M, Mp, il_kf, il_vals)
  switch (g) {
    case 1: SSK(1); break;
    case 2: SSK(2); break;
    case 4: SSK(4); break;
    default: SSK(8);
  }
#undef SSK
  ALTO_LAUNCH_CHECK("sums_stream_kernel");
  return ALTO_OK;
}

int alto_memo_fused_stream(const uint32_t *rows, const uint32_t *jcrd, const uint32_t *kcrd, const double *vals,
                           int64_t M, int32_t rank, uint32_t *il_rows, uint32_t *il_jf, uint32_t *il_k,
                           double *il_vals, void *stream) {
  ALTO_REQUIRE(M >= 0, ALTO_ERR_VALUE, "negative nnz");
  ALTO_REQUIRE(rank >= 1 && rank <= kMaxRankChunk, ALTO_ERR_UNSUPPORTED, "the fused producer supports rank <= %d",
               kMaxRankChunk);
  const int g = sums_group(rank);
  const int64_t Mp = il_len(M < 1 ? 1 : M, g);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t blocks = ceil_div(Mp, 256);
  if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
#define FSK(GV)                                                                                          \
  fused_stream_kernel<GV><<<(int)blocks, 256, 0, st>>>(rows, jcrd, kcrd, vals, M, Mp, il_rows, il_jf, il_k, \
                                                       il_vals)
  switch (g) {
    case 1: FSK(1); break;
    case 2: FSK(2); break;
    case 4: FSK(4); break;
    default: FSK(8);
  }
#undef FSK
  ALTO_LAUNCH_CHECK("fused_stream_kernel");
  return ALTO_OK;
}

int alto_memo_fused(const uint32_t *il_rows, const uint32_t *il_jf, const uint32_t *il_k, const double *il_vals,
                    int64_t M, const double *Aj, int64_t ldj, const double *Ak, int64_t ldk, int32_t rank,
                    const uint32_t *pbase, double *T, int64_t ldT, double *out, int64_t ldo, void *stream) {
  ALTO_REQUIRE(rank >= 1 && rank <= kMaxRankChunk, ALTO_ERR_UNSUPPORTED, "the fused producer supports rank <= %d",
               kMaxRankChunk);
  ALTO_REQUIRE(T == nullptr || (pbase != nullptr && ldT >= rank && (ldT & 3) == 0), ALTO_ERR_VALUE,
               "T rows must be padded to 4 columns");
  if (M == 0) return ALTO_OK;
  FusedArgs a;
  a.rows = il_rows;
  a.jf = il_jf;
  a.kc = il_k;
  a.vals = il_vals;
  a.M = M;
  const int g = sums_group(rank);
  a.Mp = il_len(M, g);
  a.Aj = Aj;
  a.ldj = ldj;
  a.Ak = Ak;
  a.ldk = ldk;
  a.rank = rank;
  a.pbase = pbase;
  a.T = T;
  a.ldT = ldT;
  a.out = out;
  a.ldo = ldo;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = (int)ceil_div(ceil_div(M, kDvSeg) * g, 256);
  const int bytes = kFusedWarp * 8;
#define FUS(GV)                                                                                        \
  {                                                                                                    \
    static bool attr = false;                                                                          \
    if (!attr) {                                                                                       \
      cudaFuncSetAttribute(memo_fused_kernel<GV>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes); \
      attr = true;                                                                                     \
    }                                                                                                  \
    memo_fused_kernel<GV><<<grid, 256, bytes, st>>>(a);                                                \
  }
  switch (g) {
    case 1: FUS(1) break;
    case 2: FUS(2) break;
    case 4: FUS(4) break;
    default: FUS(8)
  }
#undef FUS
  ALTO_LAUNCH_CHECK("memo_fused_kernel");
  return ALTO_OK;
}

int alto_memo_sums_fast(const uint32_t *il_kf, const double *il_vals, int64_t M, const uint32_t *pbase,
                        const double *Ak, int64_t ldk, int32_t rank, double *T, int64_t ldT, void *stream) {
  ALTO_REQUIRE(rank >= 1 && rank <= kMaxRankChunk, ALTO_ERR_UNSUPPORTED, "piece sums support rank <= %d",
               kMaxRankChunk);
  ALTO_REQUIRE(ldT >= rank && (ldT & 3) == 0, ALTO_ERR_VALUE, "T rows must be padded to 4 columns");
  if (M == 0) return ALTO_OK;
  SumsArgs a;
  a.kf = il_kf;
  a.vals = il_vals;
  a.M = M;
  const int g = sums_group(rank);
  a.Mp = il_len(M, g);
  a.Ak = Ak;
  a.ldk = ldk;
  a.rank = rank;
  a.pbase = pbase;
  a.T = T;
  a.ldT = ldT;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = (int)ceil_div(ceil_div(M, kDvSeg) * g, 256);
  const int bytes = kSumsWarp * 8;
#define SUMS(GV)                                                                                      \
  {                                                                                                   \
    static bool attr = false;                                                                         \
    if (!attr) {                                                                                      \
      cudaFuncSetAttribute(memo_sums_kernel<GV>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes); \
      attr = true;                                                                                    \
    }                                                                                                 \
    memo_sums_kernel<GV><<<grid, 256, bytes, st>>>(a);                                                \
  }
  switch (g) {
    case 1: SUMS(1) break;
    case 2: SUMS(2) break;
    case 4: SUMS(4) break;
    default: SUMS(8)
  }
#undef SUMS
  ALTO_LAUNCH_CHECK("memo_sums_kernel");
  return ALTO_OK;
}

}  // extern "C"
