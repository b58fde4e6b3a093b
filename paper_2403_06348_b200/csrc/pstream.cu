// Streamed-Pi Phi for the CP-APR inner loop.
//
// Inside one mode's inner loop of cp_apr_mu (pkg/src/alto/cpd/apr.py:290-310)
// only B (the scaled factor of that mode) changes; the Khatri-Rao rows
// Pi[x] = prod_{m != n} A_m[i_m] are fixed. The reference materialises them
// (PRE, precompute_krp_rows, apr.py:101-111) only when its CPU cache
// heuristic says so (select_krp_memory_mode, apr.py:188-197: never for the
// BASELINE configs). On B200 the on-the-fly Phi is bound by the L2 -> L1
// factor-row gathers (~7 TB/s of 128-byte misses), while HBM streams at
// ~6.5 TB/s with no locality needed, so here the first inner iteration runs
// the gathering kernel (dview3 Phi) and stores Pi as a side effect, and
// every later iteration streams Pi instead of gathering:
//
//   per nonzero: R doubles of Pi + u32 row + f64 value, read once, coalesced.
//
// Layout ("lane-interleaved"): the decoded view's 512-nonzero segments are
// grouped in blocks of 32 (one warp: lane = segment % 32). Slot (block, j,
// lane) holds nonzero j of segment 32*block + lane; rows/values are stored
// at slot, Pi column c at (block*512 + j)*R*32 + c*32 + lane. A warp reads
// 32 consecutive slots per load (128 or 256 contiguous bytes), and each lane
// walks its own segment in view order, so row runs are privatised in
// registers exactly like dview3 (first/last run of a lane's chunk reduced
// with fp64 atomics, the rest stored).
//
// Arithmetic per nonzero (same operations as dview3's Phi, apr.py:114-180):
//   d = max(<B[row], Pi[x]>, eps), w = v / d, Phi[row] += w * Pi[x]
// with the dot product accumulated sequentially over the columns (dview3
// sums per-lane partials with a shuffle tree), so the two differ by
// rounding only (<= 1e-12 relative in the tests).
#include <stdlib.h>
#include <string.h>

#include "alto_common.cuh"
#include "tma.cuh"

namespace alto {

namespace {

constexpr int kSeg = 512;   // decoded-view segment (dview_kernels.cu kDvSeg)
#ifndef PS_CHUNK
#define PS_CHUNK 128
#endif
constexpr int kChunk = PS_CHUNK;  // nonzeros of its segment one lane walks per launch unit

__host__ __device__ inline int64_t pstream_blocks(int64_t M) { return ((M + kSeg - 1) / kSeg + 31) / 32; }

__global__ void pstream_build_kernel(const uint32_t *__restrict__ rows, const double *__restrict__ vals,
                                     int64_t M, int64_t slots, uint32_t *__restrict__ il_rows,
                                     double *__restrict__ il_vals) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < slots;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lane = x & 31, j = (x >> 5) % kSeg, blk = (x >> 5) / kSeg;
    const int64_t v = (blk * 32 + lane) * kSeg + j;
    const bool in = v < M;
    il_rows[x] = in ? rows[v] : 0u;
    il_vals[x] = in ? vals[v] : 0.0;
  }
}

__global__ void pstream_build_compact_kernel(const uint32_t *__restrict__ rows, const double *__restrict__ vals,
                                             int64_t M, int64_t slots, uint16_t *__restrict__ il_rows,
                                             uint8_t *__restrict__ il_vals) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < slots;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lane = x & 31, j = (x >> 5) % kSeg, blk = (x >> 5) / kSeg;
    const int64_t v = (blk * 32 + lane) * kSeg + j;
    const bool in = v < M;
    il_rows[x] = in ? (uint16_t)rows[v] : (uint16_t)0;
    il_vals[x] = in ? (uint8_t)vals[v] : (uint8_t)0;
  }
}

__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_stream_f64(const double *p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

struct PstreamArgs {
  const uint32_t *rows;  // interleaved
  const double *vals;    // interleaved
  const double *pi;      // interleaved column planes
  int64_t M;
  int64_t nblk;
  int32_t rank;
  int32_t reduce_all;
  const double *scaled;
  int64_t lds;
  double eps;
  double *out;
  int64_t ldo;
  const int32_t *skip;
  int32_t compact;  // u16 rows, u8 values (phi_pstream_tma_kernel CMP)
};

// one warp = (block of 32 segments, 128-nonzero chunk of each); RP >= rank
template <int RP>
__global__ void __launch_bounds__(256) phi_pstream_kernel(const __grid_constant__ PstreamArgs a) {
  if (a.skip != nullptr && *reinterpret_cast<volatile const int32_t *>(a.skip)) return;
  constexpr int U = 2;  // nonzeros per lane in flight
  constexpr int NCH = kSeg / kChunk;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t blk = gw / NCH;
  if (blk >= a.nblk) return;
  const int j0 = (int)(gw % NCH) * kChunk;
  const int64_t seg = blk * 32 + lane;
  const int64_t cnt64 = a.M - seg * kSeg;
  const int cnt = cnt64 <= 0 ? 0 : (cnt64 >= kSeg ? kSeg : (int)cnt64);
  const int j1 = cnt < j0 + kChunk ? cnt : j0 + kChunk;  // this lane's end
  int jmax = j1;
#pragma unroll
  for (int o = 16; o; o >>= 1) jmax = max(jmax, __shfl_xor_sync(0xffffffffu, jmax, o));
  const int R = a.rank;

  constexpr uint32_t kNone = 0xffffffffu;
  uint32_t cur = kNone;
  int run_no = 0;
  double acc[RP], brow[RP];
#pragma unroll
  for (int c = 0; c < RP; ++c) acc[c] = brow[c] = 0.0;

  auto flush = [&](bool last) {
    const bool edge = a.reduce_all || run_no == 0 || last;
    double *o = a.out + (int64_t)cur * a.ldo;
#pragma unroll
    for (int c = 0; c < RP; ++c) {
      if (c < R) {
        if (edge) red_add_f64(o + c, acc[c]);
        else o[c] = acc[c];
      }
    }
  };

  const int64_t slot0 = (blk * kSeg) * 32 + lane;
  const int64_t cstride = 32;           // column plane stride (doubles)
  const int64_t jstride = (int64_t)R * 32;  // Pi doubles per j
  for (int j = j0; j < jmax; j += U) {
    uint32_t row[U];
    double v[U], p[U][RP];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t sl = slot0 + (int64_t)(j + u) * 32;  // in bounds: slots cover whole blocks
      row[u] = ld_stream_u32(a.rows + sl);
      v[u] = ld_stream_f64(a.vals + sl);
      const double *pp = a.pi + (blk * kSeg + j + u) * jstride + lane;
#pragma unroll
      for (int c = 0; c < RP; ++c) p[u][c] = c < R ? ld_stream_f64(pp + c * cstride) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (j + u < j1) {
        if (row[u] != cur) {
          if (cur != kNone) {
            flush(false);
            ++run_no;
          }
          cur = row[u];
          const double *bp = a.scaled + (int64_t)cur * a.lds;
#pragma unroll
          for (int c = 0; c < RP; ++c) {
            brow[c] = c < R ? __ldg(bp + c) : 0.0;
            acc[c] = 0.0;
          }
        }
        double d = 0.0;
#pragma unroll
        for (int c = 0; c < RP; ++c) d = fma(brow[c], p[u][c], d);
        if (d < a.eps) d = a.eps;
        const double w = v[u] / d;
#pragma unroll
        for (int c = 0; c < RP; ++c) acc[c] = fma(w, p[u][c], acc[c]);
      }
    }
  }
  if (cur != kNone) flush(true);
}

// ---- TMA-staged variant ---------------------------------------------------
// Same work unit and arithmetic; each warp streams its rows/values/Pi for JB
// j-steps at a time into shared memory with three 1D bulk copies
// (cp.async.bulk, issued by lane 0, completion on a per-warp mbarrier),
// double-buffered, so the bytes in flight do not live in registers.


#ifndef PS_WARPS
#define PS_WARPS 16
#endif
#ifndef PS_STAGES
#define PS_STAGES 2
#endif
#ifndef PS_SMEM_KB
#define PS_SMEM_KB 200
#endif
#ifndef PS_MINB
#define PS_MINB 1
#endif
constexpr int kTmaWarps = PS_WARPS;
constexpr int kTmaStages = PS_STAGES;

// LL: Poisson log-likelihood data term instead of Phi (scaled = lambda o
// A_mode, d = <scaled[row], Pi[x]> = mhat): each warp sums v * log(mhat)
// over its units into partials[1 + warp] (a.out), no output rows.
// CMP: the compact slot layout (u16 rows, u8 values: every value an integer
// in [0, 255] and the mode < 65536 rows -- CP-APR's count tensors), 83
// instead of 92 bytes per nonzero at R = 10; the same arithmetic (a u8 count
// converts to the same double).
template <int RP, int JB, bool LL = false, bool CMP = false>
__global__ void __launch_bounds__(kTmaWarps * 32, PS_MINB) phi_pstream_tma_kernel(const __grid_constant__ PstreamArgs a) {
  // Persistent warps: warp w takes work units w, w + W, w + 2W, ... (unit =
  // 32 segments x one kChunk-nonzero chunk); its stage pipeline runs across
  // unit boundaries, so no unit pays a pipeline fill. Every unit moves
  // kChunk / JB whole stages (slots cover whole blocks: in bounds).
  extern __shared__ __align__(128) unsigned char ps_smem[];
  __shared__ __align__(8) uint64_t bars[kTmaWarps][kTmaStages];
  if (a.skip != nullptr && *reinterpret_cast<volatile const int32_t *>(a.skip)) return;
  constexpr int NCH = kSeg / kChunk;
  constexpr int SPU = kChunk / JB;  // stages per unit
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int R = a.rank;
  const uint32_t rows_b = JB * (CMP ? 64 : 128), vals_b = JB * (CMP ? 32 : 256), pi_b = (uint32_t)(JB * R * 256);
  const uint32_t stage_b = rows_b + vals_b + pi_b;
  unsigned char *wb = ps_smem + (size_t)warp * kTmaStages * stage_b;
  const int64_t units = a.nblk * NCH;
  const int64_t W = (int64_t)gridDim.x * kTmaWarps;
  const int64_t w0 = (int64_t)blockIdx.x * kTmaWarps + warp;
  if (w0 >= units) {  // warps are independent (no CTA-wide barrier)
    if (LL && lane == 0) a.out[1 + w0] = 0.0;
    return;
  }
  const int64_t my_units = (units - w0 + W - 1) / W;
  const int64_t nst = my_units * SPU;
  double llsum = 0.0;

  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kTmaStages; ++s) mbar_init(&bars[warp][s], 1);
    fence_proxy_async();
  }
  __syncwarp();
  // flattened stage f -> unit w0 + (f / SPU) * W, stage f % SPU of it; unit u
  // starts at slot u * kChunk * 32 (blocks of NCH units are contiguous)
  auto issue = [&](int s, int64_t f) {
    const int64_t u = w0 + (f / SPU) * W;
    const int64_t js = (u * kChunk + (f % SPU) * JB);  // block*512 + j of the stage's first step
    unsigned char *d = wb + (size_t)s * stage_b;
    mbar_expect_tx(&bars[warp][s], stage_b);
    if constexpr (CMP) {
      bulk_g2s(d, reinterpret_cast<const uint16_t *>(a.rows) + js * 32, rows_b, &bars[warp][s]);
      bulk_g2s(d + rows_b, reinterpret_cast<const uint8_t *>(a.vals) + js * 32, vals_b, &bars[warp][s]);
    } else {
      bulk_g2s(d, a.rows + js * 32, rows_b, &bars[warp][s]);
      bulk_g2s(d + rows_b, a.vals + js * 32, vals_b, &bars[warp][s]);
    }
    bulk_g2s(d + rows_b + vals_b, a.pi + js * (int64_t)R * 32, pi_b, &bars[warp][s]);
  };
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kTmaStages; ++s)
      if (s < nst) issue(s, s);
  }

  constexpr uint32_t kNone = 0xffffffffu;
  uint32_t cur = kNone;
  int run_no = 0;
  int j1 = 0, jbase = 0;
  double acc[RP], brow[RP];
#pragma unroll
  for (int c = 0; c < RP; ++c) acc[c] = brow[c] = 0.0;
  auto flush = [&](bool last) {
    const bool edge = a.reduce_all || run_no == 0 || last;
    double *o = a.out + (int64_t)cur * a.ldo;
#pragma unroll
    for (int c = 0; c < RP; ++c) {
      if (c < R) {
        if (edge) red_add_f64(o + c, acc[c]);
        else o[c] = acc[c];
      }
    }
  };

  for (int64_t f = 0; f < nst; ++f) {
    const int s = (int)(f % kTmaStages);
    const int fs = (int)(f % SPU);
    if (fs == 0) {
      // a new unit: this lane's segment and its end inside the chunk
      const int64_t u = w0 + (f / SPU) * W;
      const int64_t seg = (u / NCH) * 32 + lane;
      const int j0 = (int)(u % NCH) * kChunk;
      const int64_t cnt64 = a.M - seg * kSeg;
      const int cnt = cnt64 <= 0 ? 0 : (cnt64 >= kSeg ? kSeg : (int)cnt64);
      j1 = cnt < j0 + kChunk ? cnt : j0 + kChunk;
      jbase = j0;
    }
    mbar_wait(&bars[warp][s], (uint32_t)((f / kTmaStages) & 1));
    const unsigned char *d = wb + (size_t)s * stage_b;
    const uint32_t *srows = reinterpret_cast<const uint32_t *>(d);
    const double *svals = reinterpret_cast<const double *>(d + rows_b);
    const uint16_t *srows16 = reinterpret_cast<const uint16_t *>(d);
    const uint8_t *svals8 = reinterpret_cast<const uint8_t *>(d + rows_b);
    const double *spi = reinterpret_cast<const double *>(d + rows_b + vals_b);
#pragma unroll
    for (int jj = 0; jj < JB; ++jj) {
      const int j = jbase + fs * JB + jj;
      if (j < j1) {
        const uint32_t row = CMP ? (uint32_t)srows16[jj * 32 + lane] : srows[jj * 32 + lane];
        const double v = CMP ? (double)svals8[jj * 32 + lane] : svals[jj * 32 + lane];
        double p[RP];
#pragma unroll
        for (int c = 0; c < RP; ++c) p[c] = c < R ? spi[(jj * R + c) * 32 + lane] : 0.0;
        if (row != cur) {
          if (!LL && cur != kNone) {
            flush(false);
            ++run_no;
          }
          cur = row;
          const double *bp = a.scaled + (int64_t)cur * a.lds;
#pragma unroll
          for (int c = 0; c < RP; ++c) {
            brow[c] = c < R ? __ldg(bp + c) : 0.0;
            acc[c] = 0.0;
          }
        }
        if constexpr (LL) {
          double m = 0.0;
#pragma unroll
          for (int c = 0; c < RP; ++c) m = fma(brow[c], p[c], m);
          llsum += v * log(m);
          continue;
        }
#ifdef PS_SPLIT_DOT
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int c = 0; c < RP; c += 2) {
          d0 = fma(brow[c], p[c], d0);
          if (c + 1 < RP) d1 = fma(brow[c + 1], p[c + 1], d1);
        }
        double dd = d0 + d1;
#else
        double dd = 0.0;
#pragma unroll
        for (int c = 0; c < RP; ++c) dd = fma(brow[c], p[c], dd);
#endif
        if (dd < a.eps) dd = a.eps;
        const double w = v / dd;
#pragma unroll
        for (int c = 0; c < RP; ++c) acc[c] = fma(w, p[c], acc[c]);
      }
    }
    __syncwarp();  // every lane is done reading stage s
    if (lane == 0 && f + kTmaStages < nst) {
      fence_proxy_async();
      issue(s, f + kTmaStages);
    }
    if (LL && fs == SPU - 1) {
      cur = kNone;
      continue;
    }
    if (fs == SPU - 1) {
      // end of the unit: the lane's last run may continue in the next chunk.
      // When all 32 lanes end in the same row (long rows: every segment of
      // the block inside it) their runs are summed with a fixed shuffle tree
      // and reduced once, instead of 32 fp64 reductions to one address.
      const uint32_t r0 = __shfl_sync(0xffffffffu, cur, 0);
      if (__all_sync(0xffffffffu, cur == r0 && cur != kNone)) {
        double *o = a.out + (int64_t)cur * a.ldo;
#pragma unroll
        for (int c = 0; c < RP; ++c) {
          double x = acc[c];
#pragma unroll
          for (int k = 16; k; k >>= 1) x += __shfl_xor_sync(0xffffffffu, x, k);
          if (lane == 0 && c < R) red_add_f64(o + c, x);
        }
      } else if (cur != kNone) {
        flush(true);
      }
      cur = kNone;
      run_no = 0;
    }
  }
  if constexpr (LL) {
#pragma unroll
    for (int k = 16; k; k >>= 1) llsum += __shfl_xor_sync(0xffffffffu, llsum, k);
    if (lane == 0) a.out[1 + w0] = llsum;
  }
}

// one warp, fixed order: lane l sums partials 1 + l, 1 + l + 32, ..., then a
// fixed shuffle tree (deterministic for a given grid)
__global__ void pstream_ll_total_kernel(double *partials, int64_t n) {
  const int lane = threadIdx.x & 31;
  double t = 0.0;
  for (int64_t i = 1 + lane; i <= n; i += 32) t += partials[i];
#pragma unroll
  for (int k = 16; k; k >>= 1) t += __shfl_xor_sync(0xffffffffu, t, k);
  if (lane == 0) partials[0] = t;
}

template <int RP, int JB, bool CMP>
void launch_pstream_tma(const PstreamArgs &a, cudaStream_t st) {
  const int bytes = kTmaWarps * kTmaStages * JB * ((CMP ? 96 : 384) + a.rank * 256);
  static int ctas_per_sm = 0;
  if (!ctas_per_sm) {
    cudaFuncSetAttribute(phi_pstream_tma_kernel<RP, JB, false, CMP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         PS_SMEM_KB * 1024);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas_per_sm, phi_pstream_tma_kernel<RP, JB, false, CMP>,
                                                  kTmaWarps * 32, bytes);
    if (ctas_per_sm < 1) ctas_per_sm = 1;
  }
  const int64_t units = a.nblk * (kSeg / kChunk);
  int64_t blocks = (int64_t)num_sms() * ctas_per_sm;
  const int64_t need = (units + kTmaWarps - 1) / kTmaWarps;
  if (blocks > need) blocks = need;
  phi_pstream_tma_kernel<RP, JB, false, CMP><<<(int)blocks, kTmaWarps * 32, bytes, st>>>(a);
}

template <int RP, int JB, bool CMP>
void launch_pstream_ll(const PstreamArgs &a, int64_t max_warps, cudaStream_t st) {
  const int bytes = kTmaWarps * kTmaStages * JB * ((CMP ? 96 : 384) + a.rank * 256);
  static int ctas_per_sm = 0;
  if (!ctas_per_sm) {
    cudaFuncSetAttribute(phi_pstream_tma_kernel<RP, JB, true, CMP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         PS_SMEM_KB * 1024);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas_per_sm, phi_pstream_tma_kernel<RP, JB, true, CMP>,
                                                  kTmaWarps * 32, bytes);
    if (ctas_per_sm < 1) ctas_per_sm = 1;
  }
  const int64_t units = a.nblk * (kSeg / kChunk);
  int64_t blocks = (int64_t)num_sms() * ctas_per_sm;
  const int64_t need = (units + kTmaWarps - 1) / kTmaWarps;
  if (blocks > need) blocks = need;
  if (blocks > max_warps / kTmaWarps) blocks = max_warps / kTmaWarps;
  if (blocks < 1) blocks = 1;
  phi_pstream_tma_kernel<RP, JB, true, CMP><<<(int)blocks, kTmaWarps * 32, bytes, st>>>(a);
  pstream_ll_total_kernel<<<1, 32, 0, st>>>(a.out, blocks * kTmaWarps);
}

template <int RP, bool CMP>
void launch_pstream_ll_cmp(const PstreamArgs &a, int64_t max_warps, cudaStream_t st) {
  const int per_j = (CMP ? 96 : 384) + a.rank * 256;
  const int budget = PS_SMEM_KB * 1024 / (kTmaWarps * kTmaStages);
  if (8 * per_j <= budget) launch_pstream_ll<RP, 8, CMP>(a, max_warps, st);
  else if (4 * per_j <= budget) launch_pstream_ll<RP, 4, CMP>(a, max_warps, st);
  else if (2 * per_j <= budget) launch_pstream_ll<RP, 2, CMP>(a, max_warps, st);
  else launch_pstream_ll<RP, 1, CMP>(a, max_warps, st);
}

template <int RP>
void launch_pstream_ll_rp(const PstreamArgs &a, int64_t max_warps, cudaStream_t st) {
  if (a.compact) launch_pstream_ll_cmp<RP, true>(a, max_warps, st);
  else launch_pstream_ll_cmp<RP, false>(a, max_warps, st);
}

template <int RP>
void launch_pstream(const PstreamArgs &a, cudaStream_t st) {
  static const int mode = getenv("ALTO_B200_PSTREAM_TMA") ? atoi(getenv("ALTO_B200_PSTREAM_TMA")) : 1;
  if (mode || a.compact) {
    // j-steps per stage: the largest of 8/4/2/1 whose double buffer for 8
    // warps fits 200 KB of shared memory
    const int per_j = (a.compact ? 96 : 384) + a.rank * 256;
    const int budget = PS_SMEM_KB * 1024 / (kTmaWarps * kTmaStages);
#define PST(JBV) (a.compact ? launch_pstream_tma<RP, JBV, true>(a, st) : launch_pstream_tma<RP, JBV, false>(a, st))
    if (8 * per_j <= budget) PST(8);
    else if (4 * per_j <= budget) PST(4);
    else if (2 * per_j <= budget) PST(2);
    else PST(1);
#undef PST
    return;
  }
  const int64_t warps = a.nblk * (kSeg / kChunk);
  const int64_t blocks = (warps * 32 + 255) / 256;
  phi_pstream_kernel<RP><<<(int)blocks, 256, 0, st>>>(a);
}

}  // namespace
}  // namespace alto

using namespace alto;

extern "C" {

int alto_pstream_sizes(int64_t M, int32_t rank, int64_t *host_slots, int64_t *host_pi_doubles) {
  ALTO_REQUIRE(M >= 0 && rank >= 1, ALTO_ERR_VALUE, "bad sizes");
  const int64_t slots = pstream_blocks(M) * kSeg * 32;
  *host_slots = slots;
  *host_pi_doubles = slots * rank;
  return ALTO_OK;
}

int alto_pstream_build(const uint32_t *rows, const double *vals, int64_t M, uint32_t *il_rows, double *il_vals,
                       void *stream) {
  ALTO_REQUIRE(M >= 0, ALTO_ERR_VALUE, "negative nnz");
  const int64_t slots = pstream_blocks(M) * kSeg * 32;
  if (slots == 0) return ALTO_OK;
  int64_t blocks = (slots + 255) / 256;
  if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
  pstream_build_kernel<<<(int)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(rows, vals, M, slots, il_rows,
                                                                                  il_vals);
  ALTO_LAUNCH_CHECK("pstream_build_kernel");
  return ALTO_OK;
}

int alto_pstream_build_compact(const uint32_t *rows, const double *vals, int64_t M, uint16_t *il_rows,
                               uint8_t *il_vals, void *stream) {
  ALTO_REQUIRE(M >= 0, ALTO_ERR_VALUE, "negative nnz");
  const int64_t slots = pstream_blocks(M) * kSeg * 32;
  if (slots == 0) return ALTO_OK;
  int64_t blocks = (slots + 255) / 256;
  if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
  pstream_build_compact_kernel<<<(int)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(rows, vals, M, slots,
                                                                                          il_rows, il_vals);
  ALTO_LAUNCH_CHECK("pstream_build_compact_kernel");
  return ALTO_OK;
}

int alto_phi_pstream(const uint32_t *il_rows, const double *il_vals, const double *pi_il, int64_t M, int32_t rank,
                     int32_t rows_recur, const double *scaled, int64_t lds, double eps, double *out, int64_t ldo,
                     const void *skip, void *stream) {
  return alto_phi_pstream2(il_rows, il_vals, 0, pi_il, M, rank, rows_recur, scaled, lds, eps, out, ldo, skip, stream);
}

int alto_phi_pstream2(const void *il_rows, const void *il_vals, int32_t compact, const double *pi_il, int64_t M,
                      int32_t rank, int32_t rows_recur, const double *scaled, int64_t lds, double eps, double *out,
                      int64_t ldo, const void *skip, void *stream) {
  ALTO_REQUIRE(rank >= 1 && rank <= 16, ALTO_ERR_UNSUPPORTED, "streamed-Pi Phi supports rank <= 16");
  ALTO_REQUIRE(M >= 0, ALTO_ERR_VALUE, "negative nnz");
  if (M == 0) return ALTO_OK;
  PstreamArgs a;
  a.rows = static_cast<const uint32_t *>(il_rows);
  a.vals = static_cast<const double *>(il_vals);
  a.compact = compact != 0;
  a.pi = pi_il;
  a.M = M;
  a.nblk = pstream_blocks(M);
  a.rank = rank;
  a.reduce_all = rows_recur != 0;
  a.scaled = scaled;
  a.lds = lds;
  a.eps = eps;
  a.out = out;
  a.ldo = ldo;
  a.skip = static_cast<const int32_t *>(skip);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch ((rank + 1) / 2) {
    case 1: launch_pstream<2>(a, st); break;
    case 2: launch_pstream<4>(a, st); break;
    case 3: launch_pstream<6>(a, st); break;
    case 4: launch_pstream<8>(a, st); break;
    case 5: launch_pstream<10>(a, st); break;
    case 6: launch_pstream<12>(a, st); break;
    case 7: launch_pstream<14>(a, st); break;
    default: launch_pstream<16>(a, st); break;
  }
  ALTO_LAUNCH_CHECK("phi_pstream_kernel");
  return ALTO_OK;
}

int alto_loglik_pstream_partials(int32_t *host_count) {
  // one partial per warp of a persistent grid (at most 2 CTAs per SM) + the total
  *host_count = num_sms() * 2 * kTmaWarps + 1;
  return ALTO_OK;
}

int alto_loglik_pstream(const uint32_t *il_rows, const double *il_vals, const double *pi_il, int64_t M,
                        int32_t rank, const double *scaled, int64_t lds, double *partials, int32_t partials_count,
                        void *stream) {
  return alto_loglik_pstream2(il_rows, il_vals, 0, pi_il, M, rank, scaled, lds, partials, partials_count, stream);
}

int alto_loglik_pstream2(const void *il_rows, const void *il_vals, int32_t compact, const double *pi_il, int64_t M,
                         int32_t rank, const double *scaled, int64_t lds, double *partials, int32_t partials_count,
                         void *stream) {
  ALTO_REQUIRE(rank >= 1 && rank <= 16, ALTO_ERR_UNSUPPORTED, "streamed-Pi log-likelihood supports rank <= 16");
  ALTO_REQUIRE(M > 0, ALTO_ERR_VALUE, "empty tensor");
  ALTO_REQUIRE(partials_count >= kTmaWarps + 1, ALTO_ERR_VALUE, "partials buffer too small");
  PstreamArgs a;
  memset(&a, 0, sizeof a);
  a.rows = static_cast<const uint32_t *>(il_rows);
  a.vals = static_cast<const double *>(il_vals);
  a.compact = compact != 0;
  a.pi = pi_il;
  a.M = M;
  a.nblk = pstream_blocks(M);
  a.rank = rank;
  a.scaled = scaled;
  a.lds = lds;
  a.out = partials;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t cap = partials_count - 1;
  switch ((rank + 1) / 2) {
    case 1: launch_pstream_ll_rp<2>(a, cap, st); break;
    case 2: launch_pstream_ll_rp<4>(a, cap, st); break;
    case 3: launch_pstream_ll_rp<6>(a, cap, st); break;
    case 4: launch_pstream_ll_rp<8>(a, cap, st); break;
    case 5: launch_pstream_ll_rp<10>(a, cap, st); break;
    case 6: launch_pstream_ll_rp<12>(a, cap, st); break;
    case 7: launch_pstream_ll_rp<14>(a, cap, st); break;
    default: launch_pstream_ll_rp<16>(a, cap, st); break;
  }
  ALTO_LAUNCH_CHECK("phi_pstream_tma_kernel<loglik>");
  return ALTO_OK;
}

}  // extern "C"
