// Memoised CP-ALS sweep on interleaved streams: the branch-free fused
// producer (piece sums + the producing mode's MTTKRP, or the plain
// fiber-factored MTTKRP) and the streaming consumer.
//
// The producing mode m0 of a memoised pair (memo.py) needs, per piece p = a
// run of equal (i, j) inside one 512-nonzero segment of m0's fiber view,
//   T[p] = sum_{x in p} v_x A_k[k_x]
// (the reference recomputes every MTTKRP, pkg/src/alto/cpd/als.py:84-96; this
// is the shared dimension-tree term of modes m0 and m1), and the next mode m1
// reads T back: MTTKRP_m1[j] = sum_pieces A_m0'[i] o T[p]. Pieces average
// 5-7 nonzeros on c2, so the row-run machinery of dview3 (a divergent flush
// branch per run end) ran ~54 warp instructions per nonzero step in round 2's
// producer. Here a piece start is one bit of the stream and the common path
// has no data-dependent branch: per nonzero one 256-bit gather of A_k[k],
// per piece one predicated gather of A_j[j], and the closed piece's row goes
// out with one predicated 256-bit streaming store at the slot where the
// consumer streams it (csrc/dview.cuh interleaved layout, one bulk copy per
// field and warp chunk, for both kernels).
#include "dview.cuh"

namespace alto {

namespace {

// fused stream jf field: fiber coordinate (< 2^30) | piece start | piece end
constexpr uint32_t kPieceStart = 0x80000000u, kPieceEnd = 0x40000000u, kFiberMask = 0x3fffffffu;
#ifndef FUSED_END
#define FUSED_END 1  // 1: a piece's A_j row is gathered at its last nonzero and added once per piece
#endif

constexpr int kSumsHead = 32;  // per-warp mbarriers (<= 4 stages x 8 B; keeps bulk-copy destinations 16 B aligned)

// ---- fused producer: piece sums + this mode's MTTKRP, branch-free ---------
//
// The producing mode's own MTTKRP, out_m0[i] = sum_x A_m1[j_x] o (v_x A_k[k_x]),
// is accumulated from the same products (A_m1's row gathered once per piece
// with a predicated load issued with the batch's A_k gathers, held while the
// piece lasts), so T is written once and never read back by the producer.
// Stream (interleaved): rows (u32), jf = j | piece-start << 31 (u32), k (u32),
// [pos: the piece's consumer slot (u32)], v (f64) = 20 (24) B per nonzero.
// Output rows: runs privatised in registers, written once, fp64 reductions
// for runs cut by a segment edge (dview3's scheme; the flush branch is taken
// once per row run, rows average thousands of nonzeros).
// cache hints of the fused kernel's gathers (A/B knobs): A_j rows are read
// once per piece in ascending j inside a row run
#ifndef FUSED_JHINT
#define FUSED_JHINT 1  // 0: default, 1: L1::no_allocate, 2: L1::evict_first
#endif
#ifndef FUSED_KHINT
#define FUSED_KHINT 0  // 0: default, 1: L1::evict_last, 2: L1::no_allocate, 3: L1::evict_first
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
#if FUSED_KHINT == 2
  asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3])
               : "l"(p));
#elif FUSED_KHINT == 3
  asm volatile("ld.global.nc.L1::evict_first.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3])
               : "l"(p));
#elif FUSED_KHINT == 1
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
#ifndef FUSED_MINB_PLAIN
#define FUSED_MINB_PLAIN 2
#endif
#ifndef FUSED_CARVEOUT_PLAIN
#define FUSED_CARVEOUT_PLAIN (FUSED_MINB_PLAIN >= 3 ? 58 : 43)
#endif
#ifndef FUSED_CARVEOUT
#define FUSED_CARVEOUT 43  // % of the 228 KB: the 100 KB configuration (2 CTAs), the rest L1 for the gathers
#endif
#ifndef FUSED_BLOCK
#define FUSED_BLOCK 256
#endif
#ifndef FUSED_STAGES
#define FUSED_STAGES 2
#endif
constexpr int kFusedStages = FUSED_STAGES;
// u32 fields rows, jf, NK gathered-mode coordinates (+ pos: the consumer
// slot of a starting piece), f64 values
template <bool POS, int NK = 1>
constexpr int fused_stage() {
  return kIlWarpChunk * 4 * (2 + NK + (POS ? 1 : 0)) + kIlWarpChunk * 8;
}
template <bool POS, int NK = 1>
constexpr int fused_warp() {
  return kSumsHead + fused_stage<POS, NK>() * kFusedStages;
}

struct FusedArgs {
  const uint32_t *rows;  // interleaved
  const uint32_t *jf;
  const uint32_t *kc;  // NK planes of Mp coordinates (the modes gathered per nonzero, ascending)
  const double *vals;
  int64_t M;
  int64_t Mp;
  const double *Aj;  // fiber mode's factor (one row per piece)
  int64_t ldj;
  const double *Ak[3];  // the other modes' factors (one row per nonzero each)
  int64_t ldk[3];
  int32_t rank;
  const uint32_t *pbase;
  const uint32_t *pos;  // interleaved consumer slot of each starting piece (T rows in consumer order), or null
  double *T;  // null: plain fiber-factored MTTKRP (no piece sums stored)
  int64_t ldT;
  double *out;
  int64_t ldo;
  const int32_t *pred;  // device predicate (alto_memo_fused_if): run iff (*pred != 0) == run_if; null: run
  int32_t run_if;
};

template <int G, bool POS, bool STORE, int NK = 1>
__global__ void __launch_bounds__(FUSED_BLOCK, STORE ? FUSED_MINB : FUSED_MINB_PLAIN) memo_fused_kernel(const __grid_constant__ FusedArgs a) {
  extern __shared__ __align__(16) unsigned char fu_smem[];
  constexpr int VEC = kVec, NG = 32 / G, CH = 4 * G, Q = G, S = kFusedStages, U = FUSED_U;
  constexpr int kFusedStage = fused_stage<POS, NK>();
  constexpr int kFusedWarp = fused_warp<POS, NK>();
  static_assert(!STORE || NK == 1, "piece sums: 3-mode tensors");
  // piece-end accumulation for 3 modes (c2 sweep 2.20 -> 2.16 ms); with
  // N - 2 >= 2 gathered modes the per-nonzero form keeps fewer registers
  // live (c3: 5.47 vs 5.64 ms per mode, profiles/r02_fused_end_ab.txt)
  constexpr bool kEnd = FUSED_END && NK == 1;
  constexpr uint32_t kNone = 0xffffffffu;
  if (a.pred != nullptr && ((*reinterpret_cast<volatile const int32_t *>(a.pred) != 0) != (a.run_if != 0))) return;
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
  const char *fk[NK];
  uint32_t ldkb[NK];
#pragma unroll
  for (int t = 0; t < NK; ++t) {
    fk[t] = reinterpret_cast<const char *>(a.Ak[t] + colld);
    ldkb[t] = (uint32_t)(a.ldk[t] * 8);
  }
  const char *fj = reinterpret_cast<const char *>(a.Aj + colld);
  const uint32_t ldjb = (uint32_t)(a.ldj * 8);

  const bool seg_ok = s0 < s1;
  constexpr bool store_t = STORE;  // false: the plain fiber-factored MTTKRP (no piece sums)
  double *tp = (store_t && !POS) ? a.T + ((int64_t)(seg_ok ? a.pbase[seg] : 0u) - 1) * a.ldT + colv : a.T;
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
#pragma unroll
      for (int t = 0; t < NK; ++t) bulk_g2s(st + (2 + t) * U32B, a.kc + t * a.Mp + src, U32B, &bars[slot]);
      if constexpr (POS) bulk_g2s(st + (2 + NK) * U32B, a.pos + src, U32B, &bars[slot]);
      bulk_g2s(st + (2 + NK + (POS ? 1 : 0)) * U32B, a.vals + src, kIlWarpChunk * 8, &bars[slot]);
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
    constexpr int VOFF = (2 + NK + (POS ? 1 : 0)) * kIlWarpChunk * 4;  // values field
    constexpr int POFF = (2 + NK) * kIlWarpChunk * 4;                  // pos field
#pragma unroll 1
    for (int k = 0; k < Q; ++k) {
#pragma unroll
      for (int ub = 0; ub < 4; ub += U) {
        // this batch's U nonzeros of quad k (half a quad per 64-bit shared
        // read when U = 2: the quad is not held in registers)
        constexpr int U32B = kIlWarpChunk * 4;
        static_assert(U == 2 || U == 4, "batches of 2 or 4 nonzeros");
        const int off = k * 16 * NG + grp * 16 + (U == 2 ? ub * 4 : 0);
        uint32_t rr[U], jv[U], kv[NK][U], pv[U];
        double vv[U];
        if constexpr (U == 2) {
          const uint2 r2 = *reinterpret_cast<const uint2 *>(st + off);
          const uint2 j2 = *reinterpret_cast<const uint2 *>(st + U32B + off);
          const double2 v2 = *reinterpret_cast<const double2 *>(st + VOFF + k * 32 * NG + grp * 16 + ub * 8 * NG);
          rr[0] = r2.x, rr[1] = r2.y, jv[0] = j2.x, jv[1] = j2.y;
#pragma unroll
          for (int t = 0; t < NK; ++t) {
            const uint2 k2 = *reinterpret_cast<const uint2 *>(st + (2 + t) * U32B + off);
            kv[t][0] = k2.x, kv[t][1] = k2.y;
          }
          vv[0] = v2.x, vv[1] = v2.y;
          if constexpr (POS) {
            const uint2 p2 = *reinterpret_cast<const uint2 *>(st + POFF + off);
            pv[0] = p2.x, pv[1] = p2.y;
          }
        } else {
          const uint4 r4 = *reinterpret_cast<const uint4 *>(st + off);
          const uint4 j4 = *reinterpret_cast<const uint4 *>(st + U32B + off);
          const unsigned char *sv = st + VOFF + k * 32 * NG + grp * 16;
          const double2 v01 = *reinterpret_cast<const double2 *>(sv);
          const double2 v23 = *reinterpret_cast<const double2 *>(sv + 16 * NG);
          rr[0] = r4.x, rr[1] = r4.y, rr[2] = r4.z, rr[3] = r4.w;
          jv[0] = j4.x, jv[1] = j4.y, jv[2] = j4.z, jv[3] = j4.w;
#pragma unroll
          for (int t = 0; t < NK; ++t) {
            const uint4 k4 = *reinterpret_cast<const uint4 *>(st + (2 + t) * U32B + off);
            kv[t][0] = k4.x, kv[t][1] = k4.y, kv[t][2] = k4.z, kv[t][3] = k4.w;
          }
          vv[0] = v01.x, vv[1] = v01.y, vv[2] = v23.x, vv[3] = v23.y;
          if constexpr (POS) {
            const uint4 p4 = *reinterpret_cast<const uint4 *>(st + POFF + off);
            pv[0] = p4.x, pv[1] = p4.y, pv[2] = p4.z, pv[3] = p4.w;
          }
        }
        double f[NK][U][VEC], g[U][VEC];
#pragma unroll
        for (int t = 0; t < NK; ++t)
#pragma unroll
          for (int u = 0; u < U; ++u)
            fused_load_k(reinterpret_cast<const double *>(fk[t] + (uint64_t)kv[t][u] * ldkb[t]), f[t][u]);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t jx = jv[u];
          fused_load_j(reinterpret_cast<const double *>(fj + (uint64_t)(jx & kFiberMask) * ldjb),
                       (jx & (kEnd ? kPieceEnd : kPieceStart)) != 0, g[u]);
        }
        if constexpr (kEnd) {
        // per nonzero: x = v A_k[k], T_p = x (+ T_p unless a piece starts);
        // at a piece's last nonzero (end bit) the piece is closed at once:
        // out_i += A_j[j] o T_p (A_j gathered for that nonzero) and T_p
        // streams out to its consumer slot -- no per-nonzero A_j product and
        // no A_j row carried between nonzeros. A row run restarts in the
        // rare flush branch. Padding (zeros, no flags) adds exact zeros.
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const bool np = (jv[u] & kPieceStart) != 0;
          const bool pe = (jv[u] & kPieceEnd) != 0;
          const bool nr = np && rr[u] != cur;
          if (nr) {
            if (cur != kNone) {
              flush(cur, false);
              ++run_no;
            }
#pragma unroll
            for (int q = 0; q < VEC; ++q) acc[q] = 0.0;
            cur = rr[u];
          }
          if constexpr (STORE && POS) {
            if (np) tp = a.T + (uint64_t)pv[u] * (uint64_t)a.ldT + colv;
          } else if constexpr (STORE) {
            if (np) tp += tstep;
          }
          const double kp = np ? 0.0 : 1.0;
#pragma unroll
          for (int q = 0; q < VEC; ++q) {
            double x = vv[u] * f[0][u][q];  // v prod_k A_k[k] (ascending modes)
#pragma unroll
            for (int t = 1; t < NK; ++t) x *= f[t][u][q];
            tq[q] = fma(tq[q], kp, x);
          }
          if (pe) {
#pragma unroll
            for (int q = 0; q < VEC; ++q) acc[q] = fma(g[u][q], tq[q], acc[q]);
          }
          if constexpr (STORE) st_cs_v4_if(tp, pe && lane_active, tq);
        }
        } else {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          // padding past the last nonzero is zeros without a piece-start
          // bit: it extends the open piece by exact zeros
          const bool np = (jv[u] >> 31) != 0;
          const bool nr = np && rr[u] != cur;
          // the closed piece's T row (predicated streaming store)
          if constexpr (STORE) st_cs_v4_if(tp, np && open && lane_active, tq);
          // a finished row run is flushed (rare: rows hold thousands of
          // nonzeros); the branch only reads acc and the run restarts through
          // the multiplier, so the common path moves no registers
          if (nr && cur != kNone) {
            flush(cur, false);
            ++run_no;
          }
          cur = nr ? rr[u] : cur;
          if constexpr (STORE && POS) {
            if (np) tp = a.T + (uint64_t)pv[u] * (uint64_t)a.ldT + colv;
          } else if constexpr (STORE) {
            if (np) tp += tstep;
          }
          open = open || np;
          const double kp = np ? 0.0 : 1.0, kr = nr ? 0.0 : 1.0;
#pragma unroll
          for (int q = 0; q < VEC; ++q) {
            jcur[q] = np ? g[u][q] : jcur[q];
            double x = vv[u] * f[0][u][q];  // v prod_k A_k[k] (ascending modes)
#pragma unroll
            for (int t = 1; t < NK; ++t) x *= f[t][u][q];
            if constexpr (STORE) tq[q] = fma(tq[q], kp, x);
            acc[q] = fma(acc[q], kr, jcur[q] * x);  // out_i += A_j[j] o (v A_k[k])
          }
        }
        }
      }
    }
  }
  if constexpr (STORE && !kEnd) st_cs_v4_if(tp, open && lane_active, tq);
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
      const bool end = (x % kDvSeg) == kDvSeg - 1 || x == M - 1 || r != rows[x + 1] || j != jcrd[x + 1];
      jf = j | (start ? kPieceStart : 0u) | (end ? kPieceEnd : 0u);
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

// ---- consumer: the next mode's MTTKRP from T rows stored in its order -----
//
// MTTKRP_m1[j] = sum_pieces A_m0'[i] o T[p] (memo.cu memo1_kernel reads T
// through a position -> piece index: random 128-byte HBM rows, latency-bound
// at ~4 TB/s). Here the producer stores every piece's T row at its consumer
// slot, so the consumer streams T: per warp chunk (4 pieces per group) one
// bulk copy of the T rows plus one each of the output rows (j) and gathered
// rows (i). Consumer layout (position x of the (j, i)-sorted pieces):
//   seg = x / 512, g = seg % NG, c = (x % 512) / 4, e = x % 4
//   slot = (seg / NG) * NG * 512 + c * 4 NG + g * 4 + e
// (a group's 4 pieces of a chunk are consecutive; padding repeats the last
// output row with zero T rows).
__host__ __device__ inline int64_t il_cons(int64_t x, int G) {
  const int NG = 32 / G;
  const int64_t seg = x / kDvSeg;
  const int o = (int)(x % kDvSeg);
  return (seg / NG) * ((int64_t)NG * kDvSeg) + (o >> 2) * 4 * NG + (seg % NG) * 4 + (o & 3);
}

#ifndef CONS_STAGES
#define CONS_STAGES 2
#endif
#ifndef CONS_MINB
#define CONS_MINB 2
#endif
constexpr int kConsStages = CONS_STAGES;
// a warp chunk: prow + pcrd (2 x 4 NG u32) + 4 NG T rows of <= 4 G doubles
template <int G>
constexpr int cons_idx() {
  return 2 * 16 * (32 / G);
}
template <int G>
constexpr int cons_stage() {
  return cons_idx<G>() + 4096;
}
template <int G>
constexpr int cons_warp() {
  return kSumsHead + cons_stage<G>() * kConsStages;
}

struct ConsArgs {
  const uint32_t *prow;  // consumer layout: output row (mode m1)
  const uint32_t *pcrd;  // gathered row (mode m0)
  const double *T;       // T rows at their consumer slots
  int64_t ldT;
  int64_t P;
  const double *A;
  int64_t lda;
  int32_t rank;
  double *out;
  int64_t ldo;
  const int32_t *pred;  // as FusedArgs::pred (alto_memo_consume_if)
  int32_t run_if;
};

template <int G>
__global__ void __launch_bounds__(256, CONS_MINB) memo_consume_kernel(const __grid_constant__ ConsArgs a) {
  extern __shared__ __align__(16) unsigned char co_smem[];
  constexpr int VEC = kVec, NG = 32 / G, S = kConsStages;
  constexpr int kConsIdx = cons_idx<G>(), kConsStage = cons_stage<G>(), kConsWarp = cons_warp<G>();
  constexpr uint32_t kNone = 0xffffffffu;
  if (a.pred != nullptr && ((*reinterpret_cast<volatile const int32_t *>(a.pred) != 0) != (a.run_if != 0))) return;
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int grp = lane / G;
  const int64_t seg = gtid / G;
  const int64_t s0 = seg * kDvSeg < a.P ? seg * kDvSeg : a.P;
  const int64_t s1 = s0 + kDvSeg < a.P ? s0 + kDvSeg : a.P;
  const bool seg_ok = s0 < s1;
  unsigned char *wbase = co_smem + (threadIdx.x >> 5) * kConsWarp;
  uint64_t *bars = reinterpret_cast<uint64_t *>(wbase);
  const int64_t wblk = gtid >> 5;
  const int colv = gl * VEC;
  bool colok[VEC];
#pragma unroll
  for (int q = 0; q < VEC; ++q) colok[q] = colv + q < a.rank;
  const bool lane_active = colok[0];
  const int colld = lane_active ? colv : 0;
  const char *fa = reinterpret_cast<const char *>(a.A + colld);
  const uint32_t ldab = (uint32_t)(a.lda * 8);
  const uint32_t rowb = (uint32_t)(a.ldT * 8);
  const uint32_t tbytes = 4 * NG * rowb;  // T rows of one warp chunk
  const uint32_t left_row = (seg_ok && s0 > 0) ? a.prow[il_cons(s0 - 1, G)] : kNone;
  const uint32_t right_row = (seg_ok && s1 < a.P) ? a.prow[il_cons(s1, G)] : kNone;

  uint32_t cur = kNone;
  int run_no = 0;
  double acc[VEC];
#pragma unroll
  for (int q = 0; q < VEC; ++q) acc[q] = 0.0;
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
      unsigned char *st = wbase + kSumsHead + slot * kConsStage;
      const int64_t src = wblk * (NG * kDvSeg) + (int64_t)c * 4 * NG;
      fence_proxy_async();
      mbar_expect_tx(&bars[slot], 2 * 16 * NG + tbytes);
      bulk_g2s(st, a.prow + src, 16 * NG, &bars[slot]);
      bulk_g2s(st + 16 * NG, a.pcrd + src, 16 * NG, &bars[slot]);
      bulk_g2s(st + kConsIdx, reinterpret_cast<const char *>(a.T) + src * rowb, tbytes, &bars[slot]);
    }
  };
  constexpr int NCH = kDvSeg / 4;  // chunks per segment
  const int nch = seg_ok ? NCH : 0;
  int wn = nch;
#pragma unroll
  for (int o = 16; o; o >>= 1) wn = max(wn, __shfl_xor_sync(0xffffffffu, wn, o));
  if (lane == 0) {
#pragma unroll
    for (int t = 0; t < S; ++t) mbar_init(&bars[t], 1);
    fence_proxy_async();
  }
  __syncwarp();
#pragma unroll
  for (int c = 0; c < S - 1; ++c)
    if (c < wn) issue(c, c);
  // odd groups read the two 16-byte halves of a T row in swapped order (two
  // groups share a quarter-warp and their rows are 4 rows apart)
  const bool swap = (grp & 1) != 0;
  for (int ch = 0; ch < wn; ++ch) {
    __syncwarp();
    if (ch + S - 1 < wn) issue(ch + S - 1, (ch + S - 1) % S);
    mbar_wait(&bars[ch % S], (uint32_t)((ch / S) & 1));
    const unsigned char *st = wbase + kSumsHead + (ch % S) * kConsStage;
    const uint4 r4 = *reinterpret_cast<const uint4 *>(st + grp * 16);
    const uint4 c4 = *reinterpret_cast<const uint4 *>(st + 16 * NG + grp * 16);
    const uint32_t rr[4] = {r4.x, r4.y, r4.z, r4.w};
    const uint32_t cc[4] = {c4.x, c4.y, c4.z, c4.w};
    double f[4][VEC];
#pragma unroll
    for (int e = 0; e < 4; ++e) load_row<VEC>(reinterpret_cast<const double *>(fa + (uint64_t)cc[e] * ldab), true, f[e]);
    const unsigned char *tr = st + kConsIdx + (grp * 4) * rowb + colld * 8;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const double2 h0 = *reinterpret_cast<const double2 *>(tr + e * rowb + (swap ? 16 : 0));
      const double2 h1 = *reinterpret_cast<const double2 *>(tr + e * rowb + (swap ? 0 : 16));
      const double t0 = swap ? h1.x : h0.x, t1 = swap ? h1.y : h0.y;
      const double t2 = swap ? h0.x : h1.x, t3 = swap ? h0.y : h1.y;
      const bool nr = rr[e] != cur;
      if (nr && cur != kNone) {
        flush(cur, false);
        ++run_no;
      }
      cur = rr[e];
      const double kr = nr ? 0.0 : 1.0;
      acc[0] = fma(f[e][0], t0, acc[0] * kr);
      acc[1] = fma(f[e][1], t1, acc[1] * kr);
      acc[2] = fma(f[e][2], t2, acc[2] * kr);
      acc[3] = fma(f[e][3], t3, acc[3] * kr);
    }
  }
  // groups past the last piece walked padding only: they never flush
  if constexpr (G < 32) {
    const uint32_t r0 = __shfl_sync(0xffffffffu, cur, 0);
    // every group of the warp ending in one row: one shuffle-tree sum, one
    // reduction (a hot row spanning the warp's segments)
    if (__all_sync(0xffffffffu, seg_ok && cur == r0 && cur != kNone)) {
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
  if (seg_ok && cur != kNone) flush(cur, true);
}

template <int G>
__global__ void cons_layout_kernel(const uint32_t *__restrict__ prow, const uint32_t *__restrict__ pcrd,
                                   const uint32_t *__restrict__ pid, int64_t P, int64_t Pp,
                                   uint32_t *__restrict__ oprow, uint32_t *__restrict__ opcrd,
                                   uint32_t *__restrict__ slot_of_piece) {
  const uint32_t last = prow[P - 1];
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < Pp; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t sl = il_cons(x, G);
    if (x < P) {
      oprow[sl] = prow[x];
      opcrd[sl] = pcrd[x];
      slot_of_piece[pid != nullptr ? pid[x] : (uint32_t)x] = (uint32_t)sl;
    } else {
      oprow[sl] = last;
      opcrd[sl] = 0u;
    }
  }
}

// per nonzero of m0's fiber view: the consumer slot of the piece it starts
// (0 elsewhere), interleaved like the producer stream; one warp per segment,
// 32 consecutive nonzeros per step, piece numbers by ballot prefix
template <int G>
__global__ void fused_pos_kernel(const uint32_t *__restrict__ rows, const uint32_t *__restrict__ jcrd, int64_t M,
                                 int64_t Mp, int64_t nseg, const uint32_t *__restrict__ pbase,
                                 const uint32_t *__restrict__ slot_of_piece, uint32_t *__restrict__ opos) {
  const int64_t nsegp = Mp / kDvSeg;
  const int lane = threadIdx.x & 31;
  const uint32_t below = (1u << lane) - 1u;
  for (int64_t seg = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; seg < nsegp;
       seg += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t s0 = seg * kDvSeg;
    uint32_t p = seg < nseg ? pbase[seg] : 0u;
    for (int64_t b = s0; b < s0 + kDvSeg; b += 32) {
      const int64_t x = b + lane;
      bool st = false;
      if (x < M) {
        const uint32_t r = rows[x], j = jcrd[x];
        st = x == s0 || r != rows[x - 1] || j != jcrd[x - 1];
      }
      const uint32_t m = __ballot_sync(0xffffffffu, st);
      opos[il_u32<G>(x)] = st ? slot_of_piece[p + __popc(m & below)] : 0u;
      p += __popc(m);
    }
  }
}

template <int G, bool P, bool ST, int NK>
void launch_fused(const FusedArgs &a, int grid, cudaStream_t st) {
  constexpr int bytes = fused_warp<P, NK>() * (FUSED_BLOCK / 32);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(memo_fused_kernel<G, P, ST, NK>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(memo_fused_kernel<G, P, ST, NK>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         ST ? FUSED_CARVEOUT : FUSED_CARVEOUT_PLAIN);
    attr = true;
  }
  memo_fused_kernel<G, P, ST, NK><<<grid, FUSED_BLOCK, bytes, st>>>(a);
}

// fused stream of an N-mode fiber view: rows, jf = fiber coordinate | piece
// start << 31, the other NK = N - 2 planes (ascending modes), values
template <int G>
__global__ void fused_stream_n_kernel(const uint32_t *__restrict__ rows, const uint32_t *__restrict__ crd,
                                      int64_t crd_ld, int nplanes, int jplane, const double *__restrict__ vals,
                                      int64_t M, int64_t Mp, uint32_t *__restrict__ orows, uint32_t *__restrict__ ojf,
                                      uint32_t *__restrict__ okc, double *__restrict__ ovals) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < Mp; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pu = il_u32<G>(x);
    uint32_t r = 0u, jf = 0u;
    double v = 0.0;
    if (x < M) {
      r = rows[x];
      const uint32_t j = crd[jplane * crd_ld + x];
      const bool start = (x % kDvSeg) == 0 || r != rows[x - 1] || j != crd[jplane * crd_ld + x - 1];
      const bool end =
          (x % kDvSeg) == kDvSeg - 1 || x == M - 1 || r != rows[x + 1] || j != crd[jplane * crd_ld + x + 1];
      jf = j | (start ? kPieceStart : 0u) | (end ? kPieceEnd : 0u);
      v = vals[x];
    }
    orows[pu] = r;
    ojf[pu] = jf;
    int t = 0;
    for (int p = 0; p < nplanes; ++p) {
      if (p == jplane) continue;
      okc[t * Mp + pu] = x < M ? crd[p * crd_ld + x] : 0u;
      ++t;
    }
    ovals[il_f64<G>(x)] = v;
  }
}

// The fused stream straight from a view's sort: `skeys` are the sorted sort
// keys (row << sbits | fiber coordinate) and `perm` the source positions
// (alto::view_sort); keys and values are gathered through perm, the other
// N - 2 coordinates decoded in registers and everything written once in the
// interleaved layout -- no permuted key / value copy, no decoded view
// (gather + decode + interleave were three passes, 4.3 of the 9.3 ms of a
// c2 stream build; profiles/r02_build_fused.txt). Bit-identical output.
template <int KW, int G>
__global__ void fused_stream_build_kernel(const __grid_constant__ Layout L, const uint64_t *__restrict__ skeys,
                                          const int64_t *__restrict__ perm, const uint64_t *__restrict__ keys,
                                          const double *__restrict__ vals, int64_t M, int64_t Mp, int mode, int fmode,
                                          int sbits, uint32_t *__restrict__ orows, uint32_t *__restrict__ ojf,
                                          uint32_t *__restrict__ okc, double *__restrict__ ovals,
                                          uint32_t *__restrict__ vrows, uint32_t *__restrict__ vfib) {
  // one thread per quad of consecutive nonzeros: a quad is 16 contiguous
  // bytes of every u32 field and two 16-byte pieces of the values in the
  // interleaved layout (vector stores), and its 4 key + 4 value gathers are
  // independent (issued together)
  const uint64_t jmask = (1ull << sbits) - 1ull;
  const int64_t nq = Mp / 4;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x0 = 4 * q;
    uint64_t sk[6];  // sort keys x0 - 1 .. x0 + 4 (neighbours decide piece starts and ends)
#pragma unroll
    for (int e = 0; e < 6; ++e) {
      const int64_t x = x0 - 1 + e;
      sk[e] = (x >= 0 && x < M) ? skeys[x] : ~0ull;
    }
    int64_t p[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) p[e] = x0 + e < M ? perm[x0 + e] : 0;
    Key k[4];
    double v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      k[e] = load_key<KW>(keys, p[e]);
      v[e] = vals[p[e]];
    }
    uint32_t r[4], jf[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t x = x0 + e;
      const bool in = x < M;
      const uint64_t s = sk[e + 1];
      const bool start = (x % kDvSeg) == 0 || s != sk[e];
      const bool end = (x % kDvSeg) == kDvSeg - 1 || x == M - 1 || s != sk[e + 2];
      r[e] = in ? (uint32_t)(s >> sbits) : 0u;
      jf[e] = in ? ((uint32_t)(s & jmask) | (start ? kPieceStart : 0u) | (end ? kPieceEnd : 0u)) : 0u;
      if (!in) v[e] = 0.0;
    }
    if (vrows != nullptr) {
      // the view's row and fiber coordinates in view order (the memoised
      // plan's piece index is built from them)
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (x0 + e < M) {
          vrows[x0 + e] = r[e];
          vfib[x0 + e] = jf[e] & kFiberMask;
        }
    }
    const int64_t pu = il_u32<G>(x0);
    *reinterpret_cast<uint4 *>(orows + pu) = make_uint4(r[0], r[1], r[2], r[3]);
    *reinterpret_cast<uint4 *>(ojf + pu) = make_uint4(jf[0], jf[1], jf[2], jf[3]);
    int t = 0;
    for (int m = 0; m < L.nmodes; ++m) {
      if (m == mode || m == fmode) continue;
      uint32_t c[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) c[e] = x0 + e < M ? (uint32_t)decode_fast<KW>(L, m, k[e]) : 0u;
      *reinterpret_cast<uint4 *>(okc + t * Mp + pu) = make_uint4(c[0], c[1], c[2], c[3]);
      ++t;
    }
    *reinterpret_cast<double2 *>(ovals + il_f64<G>(x0)) = make_double2(v[0], v[1]);
    *reinterpret_cast<double2 *>(ovals + il_f64<G>(x0 + 2)) = make_double2(v[2], v[3]);
  }
}

// ---- memo keys of the public call memo (memo.CallMemo) -----------------
// flag (preset to 1 by the caller) drops to 0 when A's first `rank` columns
// differ bitwise from the saved key (the factor a stored T was produced with)
__global__ void key_check_kernel(const double *__restrict__ A, int64_t lda, const double *__restrict__ key,
                                 int64_t ldk, int64_t rows, int rank, int32_t *flag) {
  bool diff = false;
  const int64_t total = rows * rank;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / rank;
    const int r = (int)(e - i * rank);
    diff |= __double_as_longlong(A[i * lda + r]) != __double_as_longlong(key[i * ldk + r]);
  }
  if (__any_sync(0xffffffffu, diff) && (threadIdx.x & 31) == 0) *flag = 0;
}

__global__ void key_save_kernel(const double *__restrict__ A, int64_t lda, double *__restrict__ key, int64_t ldk,
                                int64_t rows, int rank, const int32_t *pred, int save_if) {
  if (pred != nullptr && ((*reinterpret_cast<volatile const int32_t *>(pred) != 0) != (save_if != 0))) return;
  const int64_t total = rows * rank;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / rank;
    const int r = (int)(e - i * rank);
    key[i * ldk + r] = A[i * lda + r];
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

int alto_memo_fused_if(const uint32_t *il_rows, const uint32_t *il_jf, const uint32_t *il_k, const double *il_vals,
                       int64_t M, const double *Aj, int64_t ldj, const double *Ak, int64_t ldk, int32_t rank,
                       const uint32_t *pbase, const uint32_t *il_pos, double *T, int64_t ldT, double *out,
                       int64_t ldo, const int32_t *pred, int32_t run_if, void *stream) {
  ALTO_REQUIRE(rank >= 1 && rank <= kMaxRankChunk, ALTO_ERR_UNSUPPORTED, "the fused producer supports rank <= %d",
               kMaxRankChunk);
  ALTO_REQUIRE(T == nullptr || ((pbase != nullptr || il_pos != nullptr) && ldT >= rank && (ldT & 3) == 0),
               ALTO_ERR_VALUE, "T rows must be padded to 4 columns");
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
  a.Ak[0] = Ak;
  a.ldk[0] = ldk;
  a.rank = rank;
  a.pbase = pbase;
  a.pos = il_pos;
  a.T = T;
  a.ldT = ldT;
  a.out = out;
  a.ldo = ldo;
  a.pred = pred;
  a.run_if = run_if;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = (int)ceil_div(ceil_div(M, kDvSeg) * g, FUSED_BLOCK);
#define FUS(GV)                                                      \
  if (T == nullptr) launch_fused<GV, false, false, 1>(a, grid, st);  \
  else if (a.pos != nullptr) launch_fused<GV, true, true, 1>(a, grid, st); \
  else launch_fused<GV, false, true, 1>(a, grid, st);
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

int alto_memo_fused(const uint32_t *il_rows, const uint32_t *il_jf, const uint32_t *il_k, const double *il_vals,
                    int64_t M, const double *Aj, int64_t ldj, const double *Ak, int64_t ldk, int32_t rank,
                    const uint32_t *pbase, const uint32_t *il_pos, double *T, int64_t ldT, double *out, int64_t ldo,
                    void *stream) {
  return alto_memo_fused_if(il_rows, il_jf, il_k, il_vals, M, Aj, ldj, Ak, ldk, rank, pbase, il_pos, T, ldT, out,
                            ldo, nullptr, 1, stream);
}

int alto_fused_stream_n(const uint32_t *rows, const uint32_t *crd, int64_t crd_ld, int32_t nplanes, int32_t jplane,
                        const double *vals, int64_t M, int32_t rank, uint32_t *il_rows, uint32_t *il_jf,
                        uint32_t *il_k, double *il_vals, void *stream) {
  ALTO_REQUIRE(M >= 0, ALTO_ERR_VALUE, "negative nnz");
  ALTO_REQUIRE(nplanes >= 2 && nplanes <= 4 && jplane >= 0 && jplane < nplanes, ALTO_ERR_UNSUPPORTED,
               "the fused fiber stream supports 3-5 modes");
  ALTO_REQUIRE(rank >= 1 && rank <= kMaxRankChunk, ALTO_ERR_UNSUPPORTED, "rank <= %d", kMaxRankChunk);
  const int g = sums_group(rank);
  const int64_t Mp = il_len(M < 1 ? 1 : M, g);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t blocks = ceil_div(Mp, 256);
  if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
#define FSN(GV)                                                                                                   \
  fused_stream_n_kernel<GV><<<(int)blocks, 256, 0, st>>>(rows, crd, crd_ld, nplanes, jplane, vals, M, Mp, il_rows, \
                                                         il_jf, il_k, il_vals)
  switch (g) {
    case 1: FSN(1); break;
    case 2: FSN(2); break;
    case 4: FSN(4); break;
    default: FSN(8);
  }
#undef FSN
  ALTO_LAUNCH_CHECK("fused_stream_n_kernel");
  return ALTO_OK;
}

int alto_fused_stream_build(const alto_layout_t *host_layout, const void *keys, const double *vals, int64_t M,
                            int32_t mode, int32_t fiber_mode, int32_t rank, int64_t *perm, uint32_t *il_rows,
                            uint32_t *il_jf, uint32_t *il_k, double *il_vals, uint32_t *view_rows,
                            uint32_t *view_fiber, void *scratch, size_t scratch_bytes, void *stream) {
  ALTO_REQUIRE((view_rows == nullptr) == (view_fiber == nullptr), ALTO_ERR_VALUE,
               "view_rows and view_fiber go together");
  ALTO_REQUIRE(M > 0, ALTO_ERR_VALUE, "empty tensor");
  ALTO_REQUIRE(host_layout != nullptr && host_layout->nmodes >= 3 && host_layout->nmodes <= 5 && fiber_mode >= 0 &&
                   fiber_mode < host_layout->nmodes && fiber_mode != mode,
               ALTO_ERR_UNSUPPORTED, "the fused fiber stream supports 3-5 modes and a fiber mode other than the row mode");
  ALTO_REQUIRE(rank >= 1 && rank <= kMaxRankChunk, ALTO_ERR_UNSUPPORTED, "rank <= %d", kMaxRankChunk);
  for (int m = 0; m < host_layout->nmodes; ++m)
    ALTO_REQUIRE(host_layout->dims[m] < (int64_t)kPieceEnd, ALTO_ERR_UNSUPPORTED, "fused streams need modes below 2^30");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint64_t *skeys = nullptr;
  int sbits = 0;
  int rc = alto::view_sort(host_layout, keys, M, mode, fiber_mode, -1, 0, perm, scratch, scratch_bytes, st, &skeys,
                           &sbits);
  if (rc) return rc;
  const Layout D = to_device_layout(host_layout);
  const int g = sums_group(rank);
  const int64_t Mp = il_len(M, g);
  int64_t blocks = ceil_div(Mp / 4, 256);
  if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
#define FSB(KWV, GV)                                                                                            \
  fused_stream_build_kernel<KWV, GV><<<(int)blocks, 256, 0, st>>>(D, skeys, perm, static_cast<const uint64_t *>(keys), \
                                                                  vals, M, Mp, mode, fiber_mode, sbits, il_rows, il_jf, \
                                                                  il_k, il_vals, view_rows, view_fiber)
#define FSBG(KWV)          \
  switch (g) {             \
    case 1: FSB(KWV, 1); break; \
    case 2: FSB(KWV, 2); break; \
    case 4: FSB(KWV, 4); break; \
    default: FSB(KWV, 8);  \
  }
  if (D.words == 1) {
    FSBG(1)
  } else {
    FSBG(2)
  }
#undef FSBG
#undef FSB
  ALTO_LAUNCH_CHECK("fused_stream_build_kernel");
  return ALTO_OK;
}

int alto_mttkrp_fused(const uint32_t *il_rows, const uint32_t *il_jf, const uint32_t *il_k, const double *il_vals,
                      int64_t M, int32_t nk, const double *Aj, int64_t ldj, const double *const *Ak,
                      const int64_t *ldk, int32_t rank, double *out, int64_t ldo, void *stream) {
  ALTO_REQUIRE(rank >= 1 && rank <= kMaxRankChunk, ALTO_ERR_UNSUPPORTED, "the fused MTTKRP supports rank <= %d",
               kMaxRankChunk);
  ALTO_REQUIRE(nk >= 1 && nk <= 3, ALTO_ERR_UNSUPPORTED, "the fused MTTKRP supports 3-5 modes");
  if (M == 0) return ALTO_OK;
  FusedArgs a;
  memset(&a, 0, sizeof a);
  a.rows = il_rows;
  a.jf = il_jf;
  a.kc = il_k;
  a.vals = il_vals;
  a.M = M;
  const int g = sums_group(rank);
  a.Mp = il_len(M, g);
  a.Aj = Aj;
  a.ldj = ldj;
  for (int t = 0; t < nk; ++t) {
    a.Ak[t] = Ak[t];
    a.ldk[t] = ldk[t];
  }
  a.rank = rank;
  a.out = out;
  a.ldo = ldo;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = (int)ceil_div(ceil_div(M, kDvSeg) * g, FUSED_BLOCK);
#define FNK(GV)                                                   \
  switch (nk) {                                                   \
    case 1: launch_fused<GV, false, false, 1>(a, grid, st); break; \
    case 2: launch_fused<GV, false, false, 2>(a, grid, st); break; \
    default: launch_fused<GV, false, false, 3>(a, grid, st);       \
  }
  switch (g) {
    case 1: FNK(1) break;
    case 2: FNK(2) break;
    case 4: FNK(4) break;
    default: FNK(8)
  }
#undef FNK
  ALTO_LAUNCH_CHECK("memo_fused_kernel<plain>");
  return ALTO_OK;
}

int alto_memo_consumer_length(int64_t P, int32_t rank, int64_t *host_len) {
  ALTO_REQUIRE(rank >= 1 && rank <= kMaxRankChunk, ALTO_ERR_UNSUPPORTED, "rank <= %d", kMaxRankChunk);
  *host_len = il_len(P < 1 ? 1 : P, sums_group(rank));
  return ALTO_OK;
}

int alto_memo_consumer_layout(const uint32_t *prow, const uint32_t *pcrd, const uint32_t *pid, int64_t P, int32_t rank,
                              uint32_t *il_prow, uint32_t *il_pcrd, uint32_t *slot_of_piece, void *stream) {
  ALTO_REQUIRE(P > 0 && P < (int64_t)0xffffffffll, ALTO_ERR_VALUE, "bad piece count");
  ALTO_REQUIRE(rank >= 1 && rank <= kMaxRankChunk, ALTO_ERR_UNSUPPORTED, "rank <= %d", kMaxRankChunk);
  const int g = sums_group(rank);
  const int64_t Pp = il_len(P, g);
  ALTO_REQUIRE(Pp < (int64_t)0xffffffffll, ALTO_ERR_UNSUPPORTED, "too many pieces for u32 slots");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t blocks = ceil_div(Pp, 256);
  if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
#define CLK(GV) cons_layout_kernel<GV><<<(int)blocks, 256, 0, st>>>(prow, pcrd, pid, P, Pp, il_prow, il_pcrd, slot_of_piece)
  switch (g) {
    case 1: CLK(1); break;
    case 2: CLK(2); break;
    case 4: CLK(4); break;
    default: CLK(8);
  }
#undef CLK
  ALTO_LAUNCH_CHECK("cons_layout_kernel");
  return ALTO_OK;
}

int alto_memo_fused_pos(const uint32_t *rows, const uint32_t *jcrd, int64_t M, const uint32_t *pbase,
                        const uint32_t *slot_of_piece, int32_t rank, uint32_t *il_pos, void *stream) {
  ALTO_REQUIRE(M > 0, ALTO_ERR_VALUE, "empty tensor");
  ALTO_REQUIRE(rank >= 1 && rank <= kMaxRankChunk, ALTO_ERR_UNSUPPORTED, "rank <= %d", kMaxRankChunk);
  const int g = sums_group(rank);
  const int64_t Mp = il_len(M, g);
  const int64_t nseg = ceil_div(M, kDvSeg);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int blocks = (int)ceil_div(Mp / kDvSeg, 8);  // one warp per segment
  if (blocks > num_sms() * 16) blocks = num_sms() * 16;
#define FPK(GV) fused_pos_kernel<GV><<<blocks, 256, 0, st>>>(rows, jcrd, M, Mp, nseg, pbase, slot_of_piece, il_pos)
  switch (g) {
    case 1: FPK(1); break;
    case 2: FPK(2); break;
    case 4: FPK(4); break;
    default: FPK(8);
  }
#undef FPK
  ALTO_LAUNCH_CHECK("fused_pos_kernel");
  return ALTO_OK;
}

int alto_memo_consume_if(const uint32_t *il_prow, const uint32_t *il_pcrd, const double *T, int64_t ldT, int64_t P,
                         const double *A, int64_t lda, int32_t rank, double *out, int64_t ldo, const int32_t *pred,
                         int32_t run_if, void *stream) {
  ALTO_REQUIRE(rank >= 1 && rank <= kMaxRankChunk, ALTO_ERR_UNSUPPORTED, "rank <= %d", kMaxRankChunk);
  ALTO_REQUIRE(ldT >= rank && (ldT & 3) == 0 && ldT <= 4 * sums_group(rank), ALTO_ERR_VALUE,
               "T rows must be padded to 4 columns (at most 4 per lane)");
  if (P == 0) return ALTO_OK;
  ConsArgs a;
  a.prow = il_prow;
  a.pcrd = il_pcrd;
  a.T = T;
  a.ldT = ldT;
  a.P = P;
  a.A = A;
  a.lda = lda;
  a.rank = rank;
  a.out = out;
  a.ldo = ldo;
  a.pred = pred;
  a.run_if = run_if;
  const int g = sums_group(rank);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = (int)ceil_div(ceil_div(P, kDvSeg) * g, 256);
#define CON(GV)                                                                                          \
  {                                                                                                      \
    constexpr int bytes = cons_warp<GV>() * 8;                                                           \
    static bool attr = false;                                                                            \
    if (!attr) {                                                                                         \
      cudaFuncSetAttribute(memo_consume_kernel<GV>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes); \
      attr = true;                                                                                       \
    }                                                                                                    \
    memo_consume_kernel<GV><<<grid, 256, bytes, st>>>(a);                                                \
  }
  switch (g) {
    case 1: CON(1) break;
    case 2: CON(2) break;
    case 4: CON(4) break;
    default: CON(8)
  }
#undef CON
  ALTO_LAUNCH_CHECK("memo_consume_kernel");
  return ALTO_OK;
}

int alto_memo_consume(const uint32_t *il_prow, const uint32_t *il_pcrd, const double *T, int64_t ldT, int64_t P,
                      const double *A, int64_t lda, int32_t rank, double *out, int64_t ldo, void *stream) {
  return alto_memo_consume_if(il_prow, il_pcrd, T, ldT, P, A, lda, rank, out, ldo, nullptr, 1, stream);
}

int alto_memo_key_check(const double *A, int64_t lda, const double *key, int64_t ldk, int64_t rows, int32_t rank,
                        int32_t valid, int32_t *flag, void *stream) {
  ALTO_REQUIRE(rows >= 0 && rank >= 1 && lda >= rank && ldk >= rank, ALTO_ERR_VALUE, "bad key-check arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ALTO_CUDA(cudaMemsetAsync(flag, valid ? 1 : 0, sizeof(int32_t), st));
  if (!valid || rows == 0) return ALTO_OK;
  int64_t blocks = ceil_div(rows * rank, 256);
  if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
  key_check_kernel<<<(int)blocks, 256, 0, st>>>(A, lda, key, ldk, rows, rank, flag);
  ALTO_LAUNCH_CHECK("key_check_kernel");
  return ALTO_OK;
}

int alto_memo_key_save(const double *A, int64_t lda, double *key, int64_t ldk, int64_t rows, int32_t rank,
                       const int32_t *pred, int32_t save_if, void *stream) {
  ALTO_REQUIRE(rows >= 0 && rank >= 1 && lda >= rank && ldk >= rank, ALTO_ERR_VALUE, "bad key-save arguments");
  if (rows == 0) return ALTO_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t blocks = ceil_div(rows * rank, 256);
  if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
  key_save_kernel<<<(int)blocks, 256, 0, st>>>(A, lda, key, ldk, rows, rank, pred, save_if);
  ALTO_LAUNCH_CHECK("key_save_kernel");
  return ALTO_OK;
}

}  // extern "C"
