// Fast output-oriented MTTKRP / Phi over a *decoded* mode view.
//
// The reference's output-oriented strategy walks a mode-ordered copy of the
// nonzeros that stores decoded int64 coordinates (ModeOrderedView.coords,
// pkg/src/alto/partition.py:144-204). The fast path here keeps the same idea
// in a compact, B200-friendly form: per mode a copy of the ALTO stream,
// stably re-sorted by the mode coordinate, holding the row (u32), the other
// modes' coordinates (u32 each, ascending mode order; SoA) and the value.
// Measured on c2, the in-register compress decode of the 64-bit keys was a
// third of the kernel's instructions; a decoded view removes it (the stream
// stays 16-24 B/nnz).
//
// Work mapping is run_kernel's (group of G lanes per nonzero, 4 rank columns
// per lane gathered with 256-bit loads, batches of U nonzeros with all
// gathers issued before use, row runs accumulated in registers, runs cut by
// a segment edge reduced with fp64 atomics).
#include "dview.cuh"

namespace alto {

template <int NO, int G, bool PHI, bool LL = false, bool DET = false>
__global__ void __launch_bounds__(PHI ? 256 : DV3_BLOCK, PHI ? DV3_MINB_PHI : (NO == 1 ? DV3_MINB_NO1 : DV3_MINB)) dview3_kernel(const __grid_constant__ DViewArgs a) {
  extern __shared__ __align__(16) unsigned char dv3_smem[];
  if (a.skip != nullptr && *reinterpret_cast<volatile const int32_t *>(a.skip)) return;
  using SM = Dv3Smem<NO, G>;
  constexpr int S = kDv3Stages;
  constexpr int VEC = kVec;
  // nonzeros per gather batch (divides 4); Phi with 4+ modes holds more rows per nonzero
  constexpr int U = PHI ? (NO <= 2 ? DV3_UPHI : 2) : DV3_U;
  constexpr int Q = SM::Q;                   // quads per group chunk
  constexpr int CH = 4 * Q;                  // nonzeros per group chunk
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int grp = lane / G;
  const int64_t seg = gtid / G;
  const int64_t s0 = seg * kDvSeg < a.M ? seg * kDvSeg : a.M;
  const int64_t s1 = s0 + kDvSeg < a.M ? s0 + kDvSeg : a.M;
  const bool seg_ok = s0 < s1;
  unsigned char *wbase = dv3_smem + (threadIdx.x >> 5) * (S * SM::STAGE);

  const int colv = gl * VEC;
  bool colok[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) colok[v] = colv + v < a.rank;
  const bool lane_active = colok[0];
  const int colld = lane_active ? colv : 0;

  // rows are u32 (dims <= 2^32 - 1, so 0xffffffff is never a row)
  constexpr uint32_t kNone = 0xffffffffu;
  const uint32_t left_row = (seg_ok && s0 > 0) ? a.rows[s0 - 1] : kNone;
  const uint32_t right_row = (seg_ok && s1 < a.M) ? a.rows[s1] : kNone;

  // gather address = base + row * row_bytes: one IMAD.WIDE.U32 per gather
  // (factor matrices < 4 GB each)
  const char *fb[NO];
  uint32_t fldb[NO];
#pragma unroll
  for (int j = 0; j < NO; ++j) {
    fb[j] = reinterpret_cast<const char *>(a.fptr[j] + a.col0 + colld);
    fldb[j] = (uint32_t)(a.fld[j] * 8);
  }
  const char *bbase = reinterpret_cast<const char *>(a.scaled + a.col0 + colld);
  const uint32_t ldsb = (uint32_t)(a.lds * 8);

  uint32_t cur = kNone;
  double bcur[PHI ? VEC : 1] = {};  // B row of `cur` (Phi)
  double llsum = 0.0;                // LL: this group's sum of v * log(mhat)
  int run_no = 0;
  double acc[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) acc[v] = 0.0;

  auto flush = [&](uint32_t row, bool last) {
    const bool from_left = (run_no == 0) && (row == left_row), to_right = last && (row == right_row);
    const bool edge = a.reduce_all || from_left || to_right;
    if constexpr (DET) {
      if (edge) {
        det_park<VEC>(a.det, seg, from_left, to_right, row, acc, colv, gl, lane_active);
        return;
      }
    }
    if (lane_active) {
      double *o = a.out + row * a.ldo + a.col0 + colv;
      if (!edge && colok[VEC - 1] && ((a.ldo | a.col0) & 3) == 0) {
        // interior run, all 4 columns: one 256-bit store
        asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(o), "d"(acc[0]), "d"(acc[1]), "d"(acc[2]),
                     "d"(acc[3])
                     : "memory");
        return;
      }
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        if (!colok[v]) continue;
        if (edge) red_add_f64(o + v, acc[v]);
        else o[v] = acc[v];
      }
    }
  };

  // this lane's 4 nonzeros of chunk `c` -> stage slot (zero-filled past s1)
  auto issue = [&](int c, int slot) {
    if (gl >= Q) return;
    unsigned char *st = wbase + slot * SM::STAGE;
    const int64_t x = s0 + (int64_t)c * CH + 4 * gl;
    const int64_t rem = s1 - x;
    const int n = rem <= 0 ? 0 : (rem >= 4 ? 4 : (int)rem);
    const int64_t xs = n > 0 ? x : 0;
    cp_async16(st + grp * SM::GS + gl * 16, a.rows + xs, 4 * n);
#pragma unroll
    for (int j = 0; j < NO; ++j)
      cp_async16(st + (1 + j) * SM::FIELD + grp * SM::GS + gl * 16, a.crd + j * a.crd_ld + xs, 4 * n);
    unsigned char *sv = st + (1 + NO) * SM::FIELD + grp * SM::VS + gl * 32;
    cp_async16(sv, a.vals + xs, n >= 2 ? 16 : 8 * n);
    cp_async16(sv + 16, n > 2 ? a.vals + xs + 2 : a.vals + xs, n > 2 ? 8 * (n - 2) : 0);
  };

  int nch = (int)((s1 - s0 + CH - 1) / CH);
#pragma unroll
  for (int o = 16; o; o >>= 1) nch = max(nch, __shfl_xor_sync(0xffffffffu, nch, o));

#pragma unroll
  for (int c = 0; c < S - 1; ++c) {
    if (c < nch) issue(c, c);
    cp_async_commit();
  }

  for (int ch = 0; ch < nch; ++ch) {
    __syncwarp();  // every lane is done reading the slot refilled below
    if (ch + S - 1 < nch) issue(ch + S - 1, (ch + S - 1) % S);
    cp_async_commit();
    cp_async_wait<S - 1>();
    __syncwarp();  // chunk ch visible to the whole group
    const unsigned char *st = wbase + (ch % S) * SM::STAGE;
    const int64_t base = s0 + (int64_t)ch * CH;
    const int64_t rem = s1 - base;
    const int cnt = rem <= 0 ? 0 : (rem < (int64_t)CH ? (int)rem : CH);
#pragma unroll 1
    for (int k = 0; k < Q; ++k) {
      const uint4 r4 = *reinterpret_cast<const uint4 *>(st + grp * SM::GS + k * 16);
      uint4 c4[NO];
#pragma unroll
      for (int j = 0; j < NO; ++j)
        c4[j] = *reinterpret_cast<const uint4 *>(st + (1 + j) * SM::FIELD + grp * SM::GS + k * 16);
      const unsigned char *sv = st + (1 + NO) * SM::FIELD + grp * SM::VS + k * 32;
      const double2 v01 = *reinterpret_cast<const double2 *>(sv);
      const double2 v23 = *reinterpret_cast<const double2 *>(sv + 16);
#pragma unroll
      for (int ub = 0; ub < 4; ub += U) {
        uint32_t row[U];
        double vv[U];
        double f[NO][U][VEC];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = ub + u;
          row[u] = pick(r4, e);
          vv[u] = e == 0 ? v01.x : (e == 1 ? v01.y : (e == 2 ? v23.x : v23.y));
        }
        const bool pre = PHI && a.pi != nullptr;
        if (pre) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int q = 4 * k + ub + u;
            const int64_t xs = q < cnt ? base + q : 0;
            load_row<VEC>(a.pi + xs * a.ldp + a.col0 + colld, true, f[0][u]);
#pragma unroll
            for (int j = 1; j < NO; ++j)
#pragma unroll
              for (int q2 = 0; q2 < VEC; ++q2) f[j][u][q2] = 1.0;
          }
        } else {
#pragma unroll
          for (int j = 0; j < NO; ++j)
#pragma unroll
            for (int u = 0; u < U; ++u)
              load_row<VEC>(reinterpret_cast<const double *>(fb[j] + (uint64_t)pick(c4[j], ub + u) * fldb[j]), true,
                            f[j][u]);
        }
        bool same = true;  // the whole batch continues the current row
#pragma unroll
        for (int u = 0; u < U; ++u) same = same && row[u] == cur;
        // Khatri-Rao products in place (f[0] holds them), same order as v2
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int q = 0; q < VEC; ++q) {
            double t = PHI ? f[0][u][q] : vv[u] * f[0][u][q];
#pragma unroll
            for (int j = 1; j < NO; ++j) t *= f[j][u][q];
            f[0][u][q] = t;
          }
        if constexpr (PHI && !LL) {
          if (a.pi_il != nullptr && !pre) {
            // Khatri-Rao rows for the streamed-Pi Phi of the next inner
            // iterations: slot (segment block, j, lane = segment % 32), column
            // planes of 32 doubles; the 8 groups of a warp write 64
            // contiguous bytes per column
            const int64_t blk = seg >> 5;
            double *pb = a.pi_il + (blk * kDvSeg * a.rank) * 32 + (seg & 31);
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int jj = (int)(base - s0) + 4 * k + ub + u;
              if (4 * k + ub + u < cnt) {
#pragma unroll
                for (int q = 0; q < VEC; ++q)
                  if (colok[q]) {
                    // streaming store: Pi (GBs) must not evict the factor rows
                    // this kernel gathers from L2 (measured -0.04 ms per launch)
                    __stcs(pb + ((int64_t)jj * a.rank + colv + q) * 32, f[0][u][q]);
                  }
              }
            }
          }
        }
        double w[U];
        if constexpr (PHI) {
          // B rows are per output row: the run's row (bcur, inactive columns
          // zeroed at load) serves the whole batch unless a row starts in it
          double dd[U];
          if (same) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
              double d = 0.0;
#pragma unroll
              for (int q = 0; q < VEC; ++q) d = fma(bcur[q], f[0][u][q], d);
              dd[u] = d;
            }
          } else {
            double bprev[VEC];
#pragma unroll
            for (int q = 0; q < VEC; ++q) bprev[q] = bcur[q];
            uint32_t rprev = cur;
#pragma unroll
            for (int u = 0; u < U; ++u) {
              if (row[u] != rprev) {
                load_row<VEC>(reinterpret_cast<const double *>(bbase + (uint64_t)row[u] * ldsb), true, bprev);
#pragma unroll
                for (int q = 0; q < VEC; ++q) bprev[q] = colok[q] ? bprev[q] : 0.0;
                rprev = row[u];
              }
              double d = 0.0;
#pragma unroll
              for (int q = 0; q < VEC; ++q) d = fma(bprev[q], f[0][u][q], d);
              dd[u] = d;
            }
#pragma unroll
            for (int q = 0; q < VEC; ++q) bcur[q] = bprev[q];
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            double d = dd[u];
#pragma unroll
            for (int o = G / 2; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
            dd[u] = LL ? d : (d < a.eps ? a.eps : d);
          }
          if constexpr (LL) {
#pragma unroll
            for (int u = 0; u < U; ++u)
              if (gl == 0 && 4 * k + ub + u < cnt) llsum += vv[u] * log(dd[u]);
            cur = row[U - 1];  // bcur now holds this row's scaled factor row
            continue;
          }
#if DV3_DIV_SPREAD
          if constexpr (U > 1 && U <= G) {
            // every lane of the group holds all U denominators: lane gl
            // divides for nonzero gl only, then the quotients are broadcast
            // (one division per lane instead of U; same IEEE quotient)
            double dm = dd[0], vm = vv[0];
#pragma unroll
            for (int u = 1; u < U; ++u)
              if (gl == u) {
                dm = dd[u];
                vm = vv[u];
              }
            const double wm = vm / dm;
#pragma unroll
            for (int u = 0; u < U; ++u) w[u] = __shfl_sync(0xffffffffu, wm, (lane & ~(G - 1)) | u);
          } else
#endif
          {
#pragma unroll
            for (int u = 0; u < U; ++u) w[u] = vv[u] / dd[u];
          }
        }
        if (same && 4 * k + ub + U <= cnt) {
          // common case: the whole batch extends the current run -- no
          // per-nonzero run checks
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int q = 0; q < VEC; ++q)
              acc[q] = PHI ? fma(w[u], f[0][u][q], acc[q]) : acc[q] + f[0][u][q];
          continue;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const bool valid = 4 * k + ub + u < cnt;
          if constexpr (PHI) {
            if (valid) {
              if (row[u] != cur) {
                if (cur != kNone) {
                  flush(cur, false);
                  ++run_no;
                }
                cur = row[u];
#pragma unroll
                for (int q = 0; q < VEC; ++q) acc[q] = 0.0;
              }
#pragma unroll
              for (int q = 0; q < VEC; ++q) acc[q] = fma(w[u], f[0][u][q], acc[q]);
            }
          } else {
            // staged entries past the segment end are zero (value 0 -> product
            // 0), so the accumulation runs unconditionally; a new run restarts
            // it through the multiplier (acc * 1 + p == acc + p exactly), which
            // keeps the accumulators in place instead of copying them around
            // the rare run-change branch
            const bool nr = valid && row[u] != cur;
            if (nr) {
              if (cur != kNone) {
                flush(cur, false);
                ++run_no;
              }
              cur = row[u];
            }
            const double keep = nr ? 0.0 : 1.0;
#pragma unroll
            for (int q = 0; q < VEC; ++q) acc[q] = fma(acc[q], keep, f[0][u][q]);
          }
        }
      }
    }
  }
  cp_async_wait<0>();
  if constexpr (LL) {
    // fixed-order block reduction of the per-group sums -> a.out[block]
    __shared__ double wsum[32];
    double v = llsum;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) wsum[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += wsum[i];
      a.out[blockIdx.x] = t;
    }
    return;
  }
  dv3_final_flush<G, VEC, DET>(cur, acc, colok, lane_active, colv, lane, a, flush);
}

template <int NO, int G, bool PHI, bool LL = false, bool DET = false>
static void launch_dview3_one(const DViewArgs &a, int grid256, cudaStream_t st) {
  constexpr int block = PHI ? 256 : DV3_BLOCK;
  constexpr int bytes = dv3_smem_bytes<NO, G>(block);
  static bool attr = false;  // opt in above 48 KB once per instantiation
  if (!attr) {
    cudaFuncSetAttribute(dview3_kernel<NO, G, PHI, LL, DET>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    attr = true;
  }
  const int grid = (int)ceil_div((int64_t)grid256 * 256, block);
  dview3_kernel<NO, G, PHI, LL, DET><<<grid, block, bytes, st>>>(a);
}

template <int NO, int G>
static void launch_dview3_pd(const DViewArgs &a, bool phi, int grid, cudaStream_t st) {
  const bool det = a.det.val != nullptr;
  if (phi) {
    if (det) launch_dview3_one<NO, G, true, false, true>(a, grid, st);
    else launch_dview3_one<NO, G, true>(a, grid, st);
  } else {
    if (det) launch_dview3_one<NO, G, false, false, true>(a, grid, st);
    else launch_dview3_one<NO, G, false>(a, grid, st);
  }
}

__global__ void ll_total_kernel(double *partials, int n) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += partials[i];
    partials[n] = s;
  }
}

template <int NO>
static int launch_loglik_dview(const DViewArgs &a, int g, int grid, cudaStream_t st) {
  switch (g) {
    case 1: launch_dview3_one<NO, 1, true, true>(a, grid, st); break;
    case 2: launch_dview3_one<NO, 2, true, true>(a, grid, st); break;
    case 4: launch_dview3_one<NO, 4, true, true>(a, grid, st); break;
    default: launch_dview3_one<NO, 8, true, true>(a, grid, st);
  }
  ALTO_LAUNCH_CHECK("dview3_kernel<loglik>");
  ll_total_kernel<<<1, 32, 0, st>>>(a.out, grid);
  ALTO_LAUNCH_CHECK("ll_total_kernel");
  return ALTO_OK;
}

template <int NO>
static int launch_dview3(const DViewArgs &a, int g, bool phi, int grid, cudaStream_t st) {
  switch (g) {
    case 1: launch_dview3_pd<NO, 1>(a, phi, grid, st); break;
    case 2: launch_dview3_pd<NO, 2>(a, phi, grid, st); break;
    case 4: launch_dview3_pd<NO, 4>(a, phi, grid, st); break;
    default: launch_dview3_pd<NO, 8>(a, phi, grid, st);
  }
  ALTO_LAUNCH_CHECK("dview3_kernel");
  return ALTO_OK;
}

// decode a key view into rows + other-mode coordinates (SoA, u32)
template <int KW>
__global__ void decode_view_kernel(const __grid_constant__ Layout L, const uint64_t *__restrict__ keys,
                                   int64_t M, int mode, uint32_t *__restrict__ rows,
                                   uint32_t *__restrict__ crd) {
  // planes: the other modes in ascending order
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < M;
       x += (int64_t)gridDim.x * blockDim.x) {
    const Key k = load_key<KW>(keys, x);
    int j = 0;
    for (int m = 0; m < L.nmodes; ++m) {
      const uint32_t c = (uint32_t)decode_fast<KW>(L, m, k);
      if (m == mode) rows[x] = c;
      else crd[(int64_t)(j++) * crd_stride(M) + x] = c;
    }
  }
}

static int run_dview(DViewArgs a, int full_rank, bool phi, cudaStream_t st) {
  const int NO = a.nmodes - 1;
  ALTO_REQUIRE(NO >= 1 && NO <= 4, ALTO_ERR_UNSUPPORTED, "decoded-view kernels support 2..5 modes");
  for (int c0 = 0; c0 < full_rank; c0 += kMaxRankChunk) {
    a.col0 = c0;
    a.rank = full_rank - c0 < kMaxRankChunk ? full_rank - c0 : kMaxRankChunk;
    int g = 1;
    while (g * kVec < a.rank) g *= 2;
    const int grid = (int)ceil_div(ceil_div(a.M, kDvSeg) * g, 256);
    const int64_t nseg = ceil_div(a.M, kDvSeg);
    int rc;
    if (det_enabled() && !a.reduce_all && a.pi_il == nullptr) {
      rc = det_edges(nseg, &a.det, st);
      if (rc) return rc;
    } else {
      a.det = DetEdges{nullptr, nullptr, nullptr};
    }
    switch (NO) {
      case 1: rc = launch_dview3<1>(a, g, phi, grid, st); break;
      case 2: rc = launch_dview3<2>(a, g, phi, grid, st); break;
      case 3: rc = launch_dview3<3>(a, g, phi, grid, st); break;
      default: rc = launch_dview3<4>(a, g, phi, grid, st); break;
    }
    if (rc) return rc;
    if (a.det.val != nullptr) {
      rc = det_merge(a.det, nseg, a.out, a.ldo, a.col0, a.rank, st);
      if (rc) return rc;
    }
  }
  return ALTO_OK;
}



#ifndef MEMO0_FJ
#define MEMO0_FJ 1  // fiber-factored producer: the next mode's row once per piece
#endif

// Memoised CP-ALS sweep, producer side (dimension-tree reuse; no reference
// counterpart -- the reference recomputes every MTTKRP from scratch,
// pkg/src/alto/cpd/als.py:84-96). Over mode m0's decoded view sorted by
// (row i, coordinate j of the next mode m1) -- planes: JP = m1, KP = the
// remaining mode k -- a "piece" is a maximal run of equal (i, j) inside one
// 512-nonzero segment. Per nonzero q = v * A_k[k], summed per piece into
//   T[piece] = sum_{x in piece} q    (stored once per piece, for mode m1)
// and, when the piece closes, out_m0[i] += A_j[j] o T[piece] (this mode's
// MTTKRP; MEMO0_FJ: A_j gathered once per piece with a predicated load --
// MEMO0_FJ=0 gathers it per nonzero, 1.33-1.37 vs 1.25-1.30 ms on c2).
// Mode m1's MTTKRP is then out_m1[j] = sum_pieces A_m0'[i] o T[piece]
// (memo1_kernel, memo.cu), valid while A_k is unchanged -- true in the sweep
// order m0, m1, k. Staging, segments, row runs and edge reductions are
// dview3's (NO = 2, G lanes x 4 columns).
template <int G, int JP, bool DET = false>
// (no whole-quad fast path: measured faster without it, 1.65 vs 1.71 ms on c2)
__global__ void __launch_bounds__(256, DV3_MINB) memo0_kernel(const __grid_constant__ DViewArgs a) {
  constexpr int NO = 2, KP = 1 - JP;
  extern __shared__ __align__(16) unsigned char dv3_smem[];
  using SM = Dv3Smem<NO, G>;
  constexpr int S = kDv3Stages;
  constexpr int VEC = kVec;
  constexpr int U = 4;
  constexpr int Q = SM::Q;
  constexpr int CH = 4 * Q;
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int grp = lane / G;
  const int64_t seg = gtid / G;
  const int64_t s0 = seg * kDvSeg < a.M ? seg * kDvSeg : a.M;
  const int64_t s1 = s0 + kDvSeg < a.M ? s0 + kDvSeg : a.M;
  const bool seg_ok = s0 < s1;
  unsigned char *wbase = dv3_smem + (threadIdx.x >> 5) * (S * SM::STAGE);

  const int colv = gl * VEC;
  bool colok[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) colok[v] = colv + v < a.rank;
  const bool lane_active = colok[0];
  const int colld = lane_active ? colv : 0;

  constexpr uint32_t kNone = 0xffffffffu;
  const uint32_t left_row = (seg_ok && s0 > 0) ? a.rows[s0 - 1] : kNone;
  const uint32_t right_row = (seg_ok && s1 < a.M) ? a.rows[s1] : kNone;
  const char *fb[NO];
  uint32_t fldb[NO];
#pragma unroll
  for (int j = 0; j < NO; ++j) {
    fb[j] = reinterpret_cast<const char *>(a.fptr[j] + a.col0 + colld);
    fldb[j] = (uint32_t)(a.fld[j] * 8);
  }

  // pieces of this segment: T rows pbase[seg], pbase[seg] + 1, ... (the
  // consumer reads them through its position -> piece index)
  // (the kernel runs with T only: deterministic mode and rank > 32; the
  // default producer is csrc/memo_sums.cu memo_fused_kernel)
  const bool store_t = a.m_T != nullptr;
  uint32_t pcur = (seg_ok && store_t) ? a.m_pbase[seg] : 0u;  // row of the open piece (after the first open: + 1)

  uint32_t cur = kNone, curj = kNone;
  int run_no = 0;
  double acc[VEC], tq[VEC], jcur[VEC];  // jcur: A_j row of the open piece
#pragma unroll
  for (int v = 0; v < VEC; ++v) acc[v] = tq[v] = jcur[v] = 0.0;

  auto flush = [&](uint32_t row, bool last) {
    const bool from_left = (run_no == 0) && (row == left_row), to_right = last && (row == right_row);
    const bool edge = a.reduce_all || from_left || to_right;
    if constexpr (DET) {
      if (edge) {
        det_park<VEC>(a.det, seg, from_left, to_right, row, acc, colv, gl, lane_active);
        return;
      }
    }
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
  // T row of the open piece, advanced by one row per piece (a pointer add
  // per nonzero instead of an index multiply)
  const int64_t tstep = a.m_ldT;
  double *tcur = a.m_T + ((int64_t)pcur - 1) * tstep + a.col0 + colv;
  // T rows are padded to whole 32-byte sectors (ldT = padded_ld(rank)):
  // every active lane stores its 4 columns with one streaming 256-bit store
  // (columns past the rank are never read back as results)
  auto close_piece = [&]() {
    if (lane_active && store_t) {
      double *tp = tcur;
      asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(tp), "d"(tq[0]), "d"(tq[1]), "d"(tq[2]),
                   "d"(tq[3])
                   : "memory");
    }
  };

  auto issue = [&](int c, int slot) {
    if (gl >= Q) return;
    unsigned char *st = wbase + slot * SM::STAGE;
    const int64_t x = s0 + (int64_t)c * CH + 4 * gl;
    const int64_t rem = s1 - x;
    const int n = rem <= 0 ? 0 : (rem >= 4 ? 4 : (int)rem);
    const int64_t xs = n > 0 ? x : 0;
    cp_async16(st + grp * SM::GS + gl * 16, a.rows + xs, 4 * n);
#pragma unroll
    for (int j = 0; j < NO; ++j)
      cp_async16(st + (1 + j) * SM::FIELD + grp * SM::GS + gl * 16, a.crd + j * a.crd_ld + xs, 4 * n);
    unsigned char *sv = st + (1 + NO) * SM::FIELD + grp * SM::VS + gl * 32;
    cp_async16(sv, a.vals + xs, n >= 2 ? 16 : 8 * n);
    cp_async16(sv + 16, n > 2 ? a.vals + xs + 2 : a.vals + xs, n > 2 ? 8 * (n - 2) : 0);
  };

  int nch = (int)((s1 - s0 + CH - 1) / CH);
#pragma unroll
  for (int o = 16; o; o >>= 1) nch = max(nch, __shfl_xor_sync(0xffffffffu, nch, o));
#pragma unroll
  for (int c = 0; c < S - 1; ++c) {
    if (c < nch) issue(c, c);
    cp_async_commit();
  }

  for (int ch = 0; ch < nch; ++ch) {
    __syncwarp();
    if (ch + S - 1 < nch) issue(ch + S - 1, (ch + S - 1) % S);
    cp_async_commit();
    cp_async_wait<S - 1>();
    __syncwarp();
    const unsigned char *st = wbase + (ch % S) * SM::STAGE;
    const int64_t base = s0 + (int64_t)ch * CH;
    const int64_t rem = s1 - base;
    const int cnt = rem <= 0 ? 0 : (rem < (int64_t)CH ? (int)rem : CH);
#pragma unroll 1
    for (int k = 0; k < Q; ++k) {
      const uint4 r4 = *reinterpret_cast<const uint4 *>(st + grp * SM::GS + k * 16);
      uint4 c4[NO];
#pragma unroll
      for (int j = 0; j < NO; ++j)
        c4[j] = *reinterpret_cast<const uint4 *>(st + (1 + j) * SM::FIELD + grp * SM::GS + k * 16);
      const unsigned char *sv = st + (1 + NO) * SM::FIELD + grp * SM::VS + k * 32;
      const double2 v01 = *reinterpret_cast<const double2 *>(sv);
      const double2 v23 = *reinterpret_cast<const double2 *>(sv + 16);
      uint32_t row[U], jj[U];
      double vv[U];
      bool newp[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        row[u] = pick(r4, u);
        jj[u] = pick(c4[JP], u);
        vv[u] = u == 0 ? v01.x : (u == 1 ? v01.y : (u == 2 ? v23.x : v23.y));
        const uint32_t pr = u ? row[u - 1] : cur, pj = u ? jj[u - 1] : curj;
        newp[u] = (4 * k + u < cnt) && (row[u] != pr || jj[u] != pj);
      }
      double f[NO][U][VEC];
#if MEMO0_FJ
      // A_k rows for every nonzero; the next mode's row A_j only where a
      // piece starts (a predicated gather: no request for the others)
#pragma unroll
      for (int u = 0; u < U; ++u)
        load_row<VEC>(reinterpret_cast<const double *>(fb[KP] + (uint64_t)pick(c4[KP], u) * fldb[KP]), true,
                      f[KP][u]);
#pragma unroll
      for (int u = 0; u < U; ++u)
        load_row_if(reinterpret_cast<const double *>(fb[JP] + (uint64_t)jj[u] * fldb[JP]), newp[u], f[JP][u]);
#else
#pragma unroll
      for (int j = 0; j < NO; ++j)
#pragma unroll
        for (int u = 0; u < U; ++u)
          load_row<VEC>(reinterpret_cast<const double *>(fb[j] + (uint64_t)pick(c4[j], u) * fldb[j]), true, f[j][u]);
#endif
      // q = v * A_k (in f[KP]); staged entries past the segment end are
      // zeros (v = 0): they add nothing
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int q = 0; q < VEC; ++q) f[KP][u][q] = vv[u] * f[KP][u][q];
#if MEMO0_FJ
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool np = newp[u];
        const bool nr = np && row[u] != cur;
        // a piece closes where the next one starts: out_i += A_j[j] o T[p]
        // (added before a row flush: the closing piece belongs to `cur`)
        const bool close = np && curj != kNone;
        const double cp = close ? 1.0 : 0.0;
#pragma unroll
        for (int q = 0; q < VEC; ++q) acc[q] = fma(jcur[q] * cp, tq[q], acc[q]);
        st_cs_v4_if(tcur, close && lane_active && store_t, tq);
        if (nr && cur != kNone) {
          flush(cur, false);
          ++run_no;
        }
        cur = nr ? row[u] : cur;
        curj = np ? jj[u] : curj;
        tcur += np ? tstep : 0;
        const double kp = np ? 0.0 : 1.0, kr = nr ? 0.0 : 1.0;
#pragma unroll
        for (int q = 0; q < VEC; ++q) {
          tq[q] = fma(tq[q], kp, f[KP][u][q]);
          acc[q] *= kr;
          jcur[q] = np ? f[JP][u][q] : jcur[q];
        }
      }
#else
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool np = newp[u];
        const bool nr = np && row[u] != cur;  // a new row run (rare: runs are long)
        // close the open piece (predicated store); flush a finished row run
        // (the branch only reads acc, so the common path moves no
        // registers); the sums restart through the multipliers (x * 0 + y)
        st_cs_v4_if(tcur, np && curj != kNone && lane_active && store_t, tq);
        if (nr && cur != kNone) {
          flush(cur, false);
          ++run_no;
        }
        cur = nr ? row[u] : cur;
        curj = np ? jj[u] : curj;
        tcur += np ? tstep : 0;
        const double kp = np ? 0.0 : 1.0, kr = nr ? 0.0 : 1.0;
#pragma unroll
        for (int q = 0; q < VEC; ++q) {
          tq[q] = fma(tq[q], kp, f[KP][u][q]);
          acc[q] = fma(acc[q], kr, f[JP][u][q] * f[KP][u][q]);
        }
      }
#endif
    }
  }
  cp_async_wait<0>();
#if MEMO0_FJ
  if (curj != kNone) {
#pragma unroll
    for (int q = 0; q < VEC; ++q) acc[q] = fma(jcur[q], tq[q], acc[q]);
  }
#endif
  if (curj != kNone) close_piece();
  dv3_final_flush<G, VEC, DET>(cur, acc, colok, lane_active, colv, lane, a, flush);
}

template <int G, int JP, bool DET>
static void launch_memo0_det(const DViewArgs &a, int grid, cudaStream_t st) {
  constexpr int bytes = dv3_smem_bytes<2, G>(256);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(memo0_kernel<G, JP, DET>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    attr = true;
  }
  memo0_kernel<G, JP, DET><<<grid, 256, bytes, st>>>(a);
}

template <int G, int JP>
static void launch_memo0_one(const DViewArgs &a, int grid, cudaStream_t st) {
  if (a.det.val != nullptr) launch_memo0_det<G, JP, true>(a, grid, st);
  else launch_memo0_det<G, JP, false>(a, grid, st);
}

static DViewArgs dview_args(const alto_layout_t *L, const uint32_t *rows, const uint32_t *crd,
                            const double *vals, int64_t M, const alto_factors_t *F, int mode,
                            double *out, int64_t ldo) {
  DViewArgs a;
  memset(&a, 0, sizeof a);
  a.rows = rows;
  a.crd = crd;
  a.vals = vals;
  a.M = M;
  a.crd_ld = crd_stride(M);
  a.nmodes = L->nmodes;
  a.mode = mode;
  int j = 0;
  for (int m = 0; m < L->nmodes; ++m) {
    if (m == mode) continue;
    a.fptr[j] = F->ptr[m];
    a.fld[j] = F->ld[m];
    ++j;
  }
  a.out = out;
  a.ldo = ldo;
  return a;
}

static int dview_checks(const alto_layout_t *L, const alto_factors_t *F, int mode, int64_t M) {
  int rc = check_layout(L);
  if (rc) return rc;
  rc = check_factors(L, F);
  if (rc) return rc;
  ALTO_REQUIRE(mode >= 0 && mode < L->nmodes, ALTO_ERR_VALUE, "mode %d out of range for a %d-mode tensor",
               mode, L->nmodes);
  ALTO_REQUIRE(M >= 0, ALTO_ERR_VALUE, "negative nnz");
  for (int n = 0; n < L->nmodes; ++n)
    ALTO_REQUIRE(L->dims[n] <= 0xffffffffll, ALTO_ERR_UNSUPPORTED, "decoded views need dims < 2^32");
  return ALTO_OK;
}

}  // namespace alto

using namespace alto;

extern "C" {


int alto_decode_view(const alto_layout_t *host_layout, const void *view_keys, int64_t M, int32_t mode,
                     uint32_t *rows, uint32_t *crd, void *stream) {
  int rc = check_layout(host_layout);
  if (rc) return rc;
  ALTO_REQUIRE(mode >= 0 && mode < host_layout->nmodes, ALTO_ERR_VALUE, "mode %d out of range", mode);
  for (int n = 0; n < host_layout->nmodes; ++n)
    ALTO_REQUIRE(host_layout->dims[n] <= 0xffffffffll, ALTO_ERR_UNSUPPORTED, "decoded views need dims < 2^32");
  if (M <= 0) return ALTO_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Layout L = to_device_layout(host_layout);
  int64_t blocks = ceil_div(M, 256);
  if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
  if (L.words == 1)
    decode_view_kernel<1><<<(int)blocks, 256, 0, st>>>(L, static_cast<const uint64_t *>(view_keys), M, mode,
                                                       rows, crd);
  else
    decode_view_kernel<2><<<(int)blocks, 256, 0, st>>>(L, static_cast<const uint64_t *>(view_keys), M, mode,
                                                       rows, crd);
  ALTO_LAUNCH_CHECK("decode_view_kernel");
  return ALTO_OK;
}

static int run_memo0(DViewArgs a, int jp, int full_rank, cudaStream_t st) {
  int rc = ALTO_OK;
  for (int c0 = 0; c0 < full_rank; c0 += kMaxRankChunk) {
    a.col0 = c0;
    a.rank = full_rank - c0 < kMaxRankChunk ? full_rank - c0 : kMaxRankChunk;
    int g = 1;
    while (g * kVec < a.rank) g *= 2;
    const int grid = (int)ceil_div(ceil_div(a.M, kDvSeg) * g, 256);
    const int64_t nseg = ceil_div(a.M, kDvSeg);
    a.det = DetEdges{nullptr, nullptr, nullptr};
    if (det_enabled() && !a.reduce_all) {
      rc = det_edges(nseg, &a.det, st);
      if (rc) return rc;
    }
#define MEMO0(GV)                                                   \
  if (jp == 0) launch_memo0_one<GV, 0>(a, grid, st);                \
  else launch_memo0_one<GV, 1>(a, grid, st);
    switch (g) {
      case 1: MEMO0(1) break;
      case 2: MEMO0(2) break;
      case 4: MEMO0(4) break;
      default: MEMO0(8) break;
    }
#undef MEMO0
    ALTO_LAUNCH_CHECK("memo0_kernel");
    if (a.det.val != nullptr) {
      rc = det_merge(a.det, nseg, a.out, a.ldo, a.col0, a.rank, st);
      if (rc) return rc;
    }
  }
  return ALTO_OK;
}

int alto_mttkrp_memo0(const alto_layout_t *host_layout, const uint32_t *rows, const uint32_t *crd,
                      const double *vals, int64_t M, const alto_factors_t *host_factors, int32_t mode,
                      int32_t next_mode, const uint32_t *pbase, double *T, int64_t ldT,
                      double *out, int64_t ldo, void *stream) {
  int rc = dview_checks(host_layout, host_factors, mode, M);
  if (rc) return rc;
  ALTO_REQUIRE(host_layout->nmodes == 3, ALTO_ERR_UNSUPPORTED, "the memoised sweep needs a 3-mode tensor");
  ALTO_REQUIRE(next_mode >= 0 && next_mode < 3 && next_mode != mode, ALTO_ERR_VALUE, "bad next mode %d",
               next_mode);
  ALTO_REQUIRE(T != nullptr && pbase != nullptr, ALTO_ERR_VALUE, "memo0 needs the piece base and T");
  if (M == 0) return ALTO_OK;
  DViewArgs a = dview_args(host_layout, rows, crd, vals, M, host_factors, mode, out, ldo);
  a.m_pbase = pbase;
  a.m_T = T;
  a.m_ldT = ldT;
  const int jp = next_mode < mode ? next_mode : next_mode - 1;  // plane of the next mode
  return run_memo0(a, jp, host_factors->rank, static_cast<cudaStream_t>(stream));
}

int alto_mttkrp_dview(const alto_layout_t *host_layout, const uint32_t *rows, const uint32_t *crd,
                      const double *vals, int64_t M, const alto_factors_t *host_factors, int32_t mode,
                      int32_t rows_recur, int32_t fiber_plane, double *out, int64_t ldo, void *stream) {
  int rc = dview_checks(host_layout, host_factors, mode, M);
  if (rc) return rc;
  if (M == 0) return ALTO_OK;
  DViewArgs a = dview_args(host_layout, rows, crd, vals, M, host_factors, mode, out, ldo);
  a.reduce_all = rows_recur != 0;
  (void)fiber_plane;
  return run_dview(a, host_factors->rank, false, static_cast<cudaStream_t>(stream));
}

static int il_group(int rank) {
  int g = 1;
  while (g * kVec < rank) g *= 2;
  return g;
}

int alto_il_length(int64_t M, int32_t rank, int64_t *host_len) {
  ALTO_REQUIRE(M >= 0, ALTO_ERR_VALUE, "negative nnz");
  ALTO_REQUIRE(rank >= 1 && rank <= kMaxRankChunk, ALTO_ERR_UNSUPPORTED, "interleaved views support rank <= %d",
               kMaxRankChunk);
  *host_len = il_len(M < 1 ? 1 : M, il_group(rank));
  return ALTO_OK;
}

}  // extern "C"

namespace alto {
// Khatri-Rao rows of a decoded view, in view order: pi[x] = prod_{m != mode}
// A_m[i_m] in ascending mode order (the OTF multiply order, so PRE == OTF
// bitwise). A group of G lanes per nonzero, 4 columns per lane.
template <int NO, int G>
__global__ void __launch_bounds__(256) pi_dview_kernel(const __grid_constant__ DViewArgs a, double *__restrict__ pi,
                                                       int64_t ldp) {
  const int lane = threadIdx.x & 31, gl = lane & (G - 1);
  const int colv = gl * kVec;
  const bool active = colv < a.rank;
  const int colld = active ? colv : 0;
  const int64_t ngroups = (int64_t)gridDim.x * (blockDim.x / G);
  for (int64_t x = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G; x < a.M; x += ngroups) {
    double p[kVec];
#pragma unroll
    for (int j = 0; j < NO; ++j) {
      const uint32_t idx = __ldg(a.crd + j * a.crd_ld + x);
      double f[kVec];
      load_row<kVec>(a.fptr[j] + (int64_t)idx * a.fld[j] + colld, true, f);
#pragma unroll
      for (int q = 0; q < kVec; ++q) p[q] = j == 0 ? f[q] : p[q] * f[q];
    }
    if (active) {
      double *o = pi + x * ldp + colv;
#pragma unroll
      for (int q = 0; q < kVec; ++q)
        if (colv + q < a.rank) o[q] = p[q];
    }
  }
}
}  // namespace alto

extern "C" {

int alto_pi_dview(const alto_layout_t *host_layout, const uint32_t *rows, const uint32_t *crd, int64_t M,
                  const alto_factors_t *host_factors, int32_t mode, double *pi, int64_t ldp, void *stream) {
  int rc = dview_checks(host_layout, host_factors, mode, M);
  if (rc) return rc;
  if (M == 0) return ALTO_OK;
  ALTO_REQUIRE(host_factors->rank <= kMaxRankChunk, ALTO_ERR_UNSUPPORTED, "decoded-view Pi supports rank <= %d",
               kMaxRankChunk);
  const int NO = host_layout->nmodes - 1;
  ALTO_REQUIRE(NO >= 1 && NO <= 4, ALTO_ERR_UNSUPPORTED, "decoded-view kernels support 2..5 modes");
  DViewArgs a = dview_args(host_layout, rows, crd, nullptr, M, host_factors, mode, nullptr, 0);
  a.rank = host_factors->rank;
  int g = 1;
  while (g * kVec < a.rank) g *= 2;
  int64_t blocks = ceil_div(M * g, 256);
  if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
#define PI_CASE(NOV)                                                                                      \
  case NOV:                                                                                               \
    if (g == 1) pi_dview_kernel<NOV, 1><<<(int)blocks, 256, 0, st>>>(a, pi, ldp);                         \
    else if (g == 2) pi_dview_kernel<NOV, 2><<<(int)blocks, 256, 0, st>>>(a, pi, ldp);                    \
    else if (g == 4) pi_dview_kernel<NOV, 4><<<(int)blocks, 256, 0, st>>>(a, pi, ldp);                    \
    else pi_dview_kernel<NOV, 8><<<(int)blocks, 256, 0, st>>>(a, pi, ldp);                                \
    break;
  switch (NO) {
    PI_CASE(1)
    PI_CASE(2)
    PI_CASE(3)
    default:
      if (g == 1) pi_dview_kernel<4, 1><<<(int)blocks, 256, 0, st>>>(a, pi, ldp);
      else if (g == 2) pi_dview_kernel<4, 2><<<(int)blocks, 256, 0, st>>>(a, pi, ldp);
      else if (g == 4) pi_dview_kernel<4, 4><<<(int)blocks, 256, 0, st>>>(a, pi, ldp);
      else pi_dview_kernel<4, 8><<<(int)blocks, 256, 0, st>>>(a, pi, ldp);
  }
#undef PI_CASE
  ALTO_LAUNCH_CHECK("pi_dview_kernel");
  return ALTO_OK;
}

static int loglik_dview_grid(int64_t M, int rank) {
  int g = 1;
  while (g * kVec < rank) g *= 2;
  return (int)ceil_div(ceil_div(M, kDvSeg) * g, 256);
}

int alto_loglik_dview_partials(int64_t M, int32_t rank, int32_t *host_count) {
  *host_count = loglik_dview_grid(M < 1 ? 1 : M, rank) + 1;
  return ALTO_OK;
}

int alto_loglik_dview(const alto_layout_t *host_layout, const uint32_t *rows, const uint32_t *crd,
                      const double *vals, int64_t M, const alto_factors_t *host_factors, int32_t mode,
                      const double *scaled, int64_t lds, double *partials, void *stream) {
  int rc = dview_checks(host_layout, host_factors, mode, M);
  if (rc) return rc;
  ALTO_REQUIRE(M > 0, ALTO_ERR_VALUE, "empty tensor");
  ALTO_REQUIRE(host_factors->rank <= kMaxRankChunk, ALTO_ERR_UNSUPPORTED,
               "decoded-view log-likelihood supports rank <= %d", kMaxRankChunk);
  const int NO = host_layout->nmodes - 1;
  ALTO_REQUIRE(NO >= 1 && NO <= 4, ALTO_ERR_UNSUPPORTED, "decoded-view kernels support 2..5 modes");
  DViewArgs a = dview_args(host_layout, rows, crd, vals, M, host_factors, mode, partials, 0);
  a.scaled = scaled;
  a.lds = lds;
  a.eps = 0.0;
  a.rank = host_factors->rank;
  a.col0 = 0;
  int g = 1;
  while (g * kVec < a.rank) g *= 2;
  const int grid = loglik_dview_grid(M, a.rank);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (NO) {
    case 1: return launch_loglik_dview<1>(a, g, grid, st);
    case 2: return launch_loglik_dview<2>(a, g, grid, st);
    case 3: return launch_loglik_dview<3>(a, g, grid, st);
    default: return launch_loglik_dview<4>(a, g, grid, st);
  }
}

int alto_phi_dview(const alto_layout_t *host_layout, const uint32_t *rows, const uint32_t *crd,
                   const double *vals, int64_t M, const alto_factors_t *host_factors, int32_t mode,
                   int32_t rows_recur, int32_t fiber_plane, const double *scaled, int64_t lds, const double *pi,
                   int64_t ldp,
                   double eps, double *out, int64_t ldo, const void *skip, double *pi_il_out, void *stream) {
  int rc = dview_checks(host_layout, host_factors, mode, M);
  if (rc) return rc;
  if (M == 0) return ALTO_OK;
  ALTO_REQUIRE(host_factors->rank <= kMaxRankChunk, ALTO_ERR_UNSUPPORTED, "decoded-view Phi supports rank <= %d",
               kMaxRankChunk);
  ALTO_REQUIRE(pi_il_out == nullptr || (pi == nullptr && host_factors->rank <= 16), ALTO_ERR_UNSUPPORTED,
               "Pi write-out needs the on-the-fly Phi and rank <= 16");
  DViewArgs a = dview_args(host_layout, rows, crd, vals, M, host_factors, mode, out, ldo);
  a.scaled = scaled;
  a.lds = lds;
  a.pi = pi;
  a.ldp = ldp;
  a.eps = eps;
  a.skip = static_cast<const int32_t *>(skip);
  a.reduce_all = rows_recur != 0;
  a.pi_il = pi_il_out;
  (void)fiber_plane;
  return run_dview(a, host_factors->rank, true, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
