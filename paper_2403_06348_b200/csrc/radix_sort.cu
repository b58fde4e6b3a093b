// Stable LSD radix sort of (key, 8-byte payload) pairs for the ALTO encoder.
//
// Replaces the reference's argsort(kind="stable") / lexsort((lo, hi))
// (pkg/src/alto/tensor.py:201-205) and the stable per-mode argsorts of the
// mode-ordered views (pkg/src/alto/partition.py:185-188). Keys are uint64 or
// {lo, hi} uint64 pairs; only the low `total_bits` bits take part, in 8-bit
// digits (c2: 43 bits -> 6 passes; 128-bit c5 keys: 95 bits -> 12 passes).
//
// B200 structure (one-sweep LSD):
//   1. one read of the keys builds the digit histograms of every pass at
//      once (shared-memory counters);
//   2. per pass, one kernel: a CTA takes the next tile of 3840 (64-bit) or
//      2560 (128-bit) keys (tile ids from
//      an atomic counter, so every predecessor is already resident), ranks its
//      keys stably with warp match/ballot (warp-striped order = input order),
//      publishes its per-digit counts and resolves its global offsets by
//      decoupled look-back over the predecessors' published counts, then
//      stages keys and payloads in shared memory in digit order so the
//      scatter to HBM is written in contiguous per-digit runs.
// Every pass moves 2 x (key + payload) bytes per element: 32 B/element for
// 64-bit keys, the HBM floor of an out-of-place LSD pass.
#include <string.h>

#include "alto_common.cuh"

namespace alto {

namespace {

constexpr int kRsThreads = 256;
constexpr int kRsWarps = kRsThreads / 32;
// keys per thread and resident CTAs per SM, by key width: the tile's keys,
// payloads and digits are staged in shared memory, and a pass is
// latency-bound (profiles/r02_ncu_radix_pass.txt), so the largest tile that
// still lets three CTAs share an SM wins (A/B in profiles/r02_radix_tile_ab.txt)
#ifndef RS_ITEMS1
#define RS_ITEMS1 15
#endif
#ifndef RS_MINB1
#define RS_MINB1 3
#endif
#ifndef RS_ITEMS2
#define RS_ITEMS2 10
#endif
#ifndef RS_MINB2
#define RS_MINB2 3
#endif
#ifndef RS_BALLOT_MATCH
#define RS_BALLOT_MATCH 1
#endif
template <int KW>
struct RsCfg {
  static constexpr int kItems = KW == 1 ? RS_ITEMS1 : RS_ITEMS2;
  static constexpr int kMinBlocks = KW == 1 ? RS_MINB1 : RS_MINB2;
  static constexpr int kTile = kRsThreads * kItems;  // keys per tile
};
constexpr int kRsBins = 256;
constexpr int kRsMaxPasses = 16;
constexpr uint32_t kFlagAggregate = 1u << 30;
constexpr uint32_t kFlagPrefix = 2u << 30;
constexpr uint32_t kCountMask = (1u << 30) - 1;

template <int KW>
struct RsKey;
template <>
struct RsKey<1> {
  uint64_t w0;
};
template <>
struct RsKey<2> {
  uint64_t w0, w1;
};

template <int KW>
__device__ __forceinline__ RsKey<KW> rs_load(const uint64_t *keys, int64_t i) {
  RsKey<KW> k;
  if constexpr (KW == 1) {
    k.w0 = keys[i];
  } else {
    const ulonglong2 v = reinterpret_cast<const ulonglong2 *>(keys)[i];
    k.w0 = v.x;
    k.w1 = v.y;
  }
  return k;
}

template <int KW>
__device__ __forceinline__ void rs_store(uint64_t *keys, int64_t i, const RsKey<KW> &k) {
  if constexpr (KW == 1) {
    keys[i] = k.w0;
  } else {
    reinterpret_cast<ulonglong2 *>(keys)[i] = make_ulonglong2(k.w0, k.w1);
  }
}

template <int KW>
__device__ __forceinline__ uint32_t rs_digit(const RsKey<KW> &k, int shift) {
  if constexpr (KW == 1) {
    return (uint32_t)(k.w0 >> shift) & 0xffu;
  } else {
    return (uint32_t)((shift < 64 ? k.w0 >> shift : k.w1 >> (shift - 64))) & 0xffu;
  }
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// all digit histograms in one read of the keys (shared-memory atomics; the
// hardware serialises only lanes that hit the same counter)
template <int KW>
__global__ void __launch_bounds__(kRsThreads) rs_hist_kernel(const uint64_t *__restrict__ keys, int64_t M,
                                                             int passes, uint32_t *__restrict__ hist) {
  __shared__ uint32_t sh[kRsMaxPasses * kRsBins];
  for (int i = threadIdx.x; i < passes * kRsBins; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < M; base += stride) {
    const int64_t i = base + threadIdx.x;
    const bool valid = i < M;
    RsKey<KW> k{};
    if (valid) k = rs_load<KW>(keys, i);
    if (valid)
      for (int p = 0; p < passes; ++p) atomicAdd(&sh[p * kRsBins + rs_digit<KW>(k, 8 * p)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kRsBins; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// exclusive scan of each pass's 256-bin histogram -> digit base offsets
__global__ void __launch_bounds__(kRsBins) rs_scan_kernel(const uint32_t *__restrict__ hist,
                                                          uint32_t *__restrict__ offsets) {
  __shared__ uint32_t warp_tot[kRsBins / 32];
  const int p = blockIdx.x;
  const int d = threadIdx.x, lane = d & 31, w = d >> 5;
  const uint32_t v = hist[p * kRsBins + d];
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  uint32_t add = 0;
  for (int i = 0; i < w; ++i) add += warp_tot[i];
  offsets[p * kRsBins + d] = add + x - v;
}

template <int KW>
struct RsSmem {
  static constexpr int kRsTile = RsCfg<KW>::kTile;
  static constexpr int kKeyBytes = kRsTile * 8 * KW;
  static constexpr int kValBytes = kRsTile * 8;
  // staging area (keys, then payloads) + the tile's payloads as loaded
  // (cp.async at kernel start) + per-position digits
  static constexpr int kBytes = kKeyBytes + kValBytes + kRsTile;
};

__device__ __forceinline__ void rs_cp_async16(void *smem, const void *gmem, int src_bytes) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(src_bytes)
               : "memory");
}

template <int KW>
__global__ void __launch_bounds__(kRsThreads, RsCfg<KW>::kMinBlocks)
    rs_pass_kernel(const uint64_t *__restrict__ kin, const uint64_t *__restrict__ vin,
                   uint64_t *__restrict__ kout, uint64_t *__restrict__ vout, int64_t M, int shift,
                   const uint32_t *__restrict__ offsets, uint32_t *status, uint32_t *tile_counter) {
  extern __shared__ __align__(16) unsigned char rs_smem[];
  constexpr int kRsItems = RsCfg<KW>::kItems, kRsTile = RsCfg<KW>::kTile;
  __shared__ uint32_t s_tile;
  __shared__ uint32_t wcnt[kRsWarps][kRsBins];  // per-warp digit counts -> exclusive offsets
  __shared__ uint32_t gbase[kRsBins];           // global base of this tile's run of digit d
  __shared__ uint32_t tstart[kRsBins];          // tile-local start of digit d
  __shared__ uint32_t warp_tot[kRsWarps];
  uint64_t *stage = reinterpret_cast<uint64_t *>(rs_smem);
  uint64_t *vbuf = reinterpret_cast<uint64_t *>(rs_smem + RsSmem<KW>::kKeyBytes);
  uint8_t *sdig = rs_smem + RsSmem<KW>::kKeyBytes + RsSmem<KW>::kValBytes;

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  for (int i = tid; i < kRsWarps * kRsBins; i += kRsThreads) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t base = (int64_t)tile * kRsTile;
  const int n = (int)(M - base < kRsTile ? M - base : kRsTile);
  // the tile's payloads start streaming into shared memory right away (no
  // registers held); they are only needed after the keys are scattered
  for (int c = tid; c < kRsTile / 2; c += kRsThreads) {
    const int e = 2 * c;  // 2 payloads per 16-byte chunk
    const int valid = n - e >= 2 ? 2 : (n - e > 0 ? n - e : 0);
    rs_cp_async16(vbuf + e, vin + base + (valid ? e : 0), 8 * valid);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");

  // load + stable warp-local ranking (item i of lane l: base + w*512 + i*32 + l)
  RsKey<KW> k[kRsItems];
  uint32_t dig[kRsItems], rnk[kRsItems];
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < kRsItems; ++i) {
    const int64_t x = base + w * (32 * kRsItems) + i * 32 + lane;
    const bool valid = x < M;
    if (valid) k[i] = rs_load<KW>(kin, x);
    dig[i] = valid ? rs_digit<KW>(k[i], shift) : kRsBins;
  }
#pragma unroll
  for (int i = 0; i < kRsItems; ++i) {
    const uint32_t d = dig[i];
#if RS_BALLOT_MATCH
    // lanes with the same digit by 9 ballots (digits 0..256) instead of MATCH.ANY
    uint32_t peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 9; ++b) {
      const bool bit = (d >> b) & 1u;
      const uint32_t vote = __ballot_sync(0xffffffffu, bit);
      peers &= bit ? vote : ~vote;
    }
#else
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
#endif
    const uint32_t before = d < kRsBins ? wcnt[w][d] : 0u;
    __syncwarp();
    if (d < kRsBins && lane == __ffs(peers) - 1) wcnt[w][d] = before + (uint32_t)__popc(peers);
    __syncwarp();
    rnk[i] = before + (uint32_t)__popc(peers & lt);
  }
  __syncthreads();

  // per digit (thread = digit): exclusive over warps, tile total
  const int d = tid;
  uint32_t total = 0;
#pragma unroll
  for (int ww = 0; ww < kRsWarps; ++ww) {
    const uint32_t c = wcnt[ww][d];
    wcnt[ww][d] = total;
    total += c;
  }
  // decoupled look-back over the predecessors' per-digit counts
  volatile uint32_t *vs = status;
  uint32_t prefix = 0;
  if (tile == 0) {
    vs[d] = kFlagPrefix | total;
  } else {
    vs[(int64_t)tile * kRsBins + d] = kFlagAggregate | total;
    for (int64_t t = (int64_t)tile - 1; t >= 0; --t) {
      uint32_t s;
      do {
        s = vs[t * kRsBins + d];
      } while ((s & ~kCountMask) == 0);
      prefix += s & kCountMask;
      if ((s & ~kCountMask) == kFlagPrefix) break;
    }
    vs[(int64_t)tile * kRsBins + d] = kFlagPrefix | (prefix + total);
  }
  gbase[d] = offsets[d] + prefix;
  // tile-local digit starts (block exclusive scan of the totals)
  uint32_t x = total;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  uint32_t add = 0;
  for (int i = 0; i < w; ++i) add += warp_tot[i];
  tstart[d] = add + x - total;
  __syncthreads();

  // stage keys in digit order, write contiguous per-digit runs
  uint32_t lpos[kRsItems];
#pragma unroll
  for (int i = 0; i < kRsItems; ++i) {
    const uint32_t dd = dig[i];
    lpos[i] = dd < kRsBins ? tstart[dd] + wcnt[w][dd] + rnk[i] : 0xffffffffu;
    if (dd < kRsBins) {
      if constexpr (KW == 1) {
        stage[lpos[i]] = k[i].w0;
      } else {
        stage[2 * lpos[i]] = k[i].w0;
        stage[2 * lpos[i] + 1] = k[i].w1;
      }
      sdig[lpos[i]] = (uint8_t)dd;
    }
  }
  __syncthreads();
  for (int j = tid; j < n; j += kRsThreads) {
    const uint32_t dd = sdig[j];
    const int64_t g = (int64_t)gbase[dd] + (j - (int)tstart[dd]);
    if constexpr (KW == 1) {
      kout[g] = stage[j];
    } else {
      RsKey<2> kk;
      kk.w0 = stage[2 * j];
      kk.w1 = stage[2 * j + 1];
      rs_store<2>(kout, g, kk);
    }
  }
  __syncthreads();
  // payloads: loaded order -> digit order through the staging area
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kRsItems; ++i)
    if (lpos[i] != 0xffffffffu) stage[lpos[i]] = vbuf[w * (32 * kRsItems) + i * 32 + lane];
  __syncthreads();
  for (int j = tid; j < n; j += kRsThreads) {
    const uint32_t dd = sdig[j];
    vout[(int64_t)gbase[dd] + (j - (int)tstart[dd])] = stage[j];
  }
}

inline size_t rs_align(size_t b) { return (b + 255) & ~size_t(255); }

}  // namespace

size_t radix_sort_scratch(int64_t M, int words) {
  const int kRsTile = words == 1 ? RsCfg<1>::kTile : RsCfg<2>::kTile;
  const int64_t tiles = (M + kRsTile - 1) / kRsTile;
  return rs_align((size_t)M * 8 * words) + rs_align((size_t)M * 8) +
         rs_align((size_t)kRsMaxPasses * kRsBins * 4 * 2) + rs_align((size_t)(tiles < 1 ? 1 : tiles) * kRsBins * 4) +
         rs_align(kRsMaxPasses * 4) + 256;
}

// Sort (keys, vals) in place by the low total_bits bits of the keys, stable.
int radix_sort_pairs(int words, int total_bits, void *keys, void *vals, int64_t M, void *scratch,
                     size_t scratch_bytes, cudaStream_t st) {
  if (M <= 1) return ALTO_OK;
  ALTO_REQUIRE(M < (int64_t)kCountMask, ALTO_ERR_UNSUPPORTED, "radix sort supports < 2^30 elements");
  ALTO_REQUIRE(scratch_bytes >= radix_sort_scratch(M, words), ALTO_ERR_VALUE, "sort scratch too small");
  const int bits = total_bits < 1 ? 1 : total_bits;
  const int passes = (bits + 7) / 8;
  ALTO_REQUIRE(passes <= kRsMaxPasses && bits <= 64 * words, ALTO_ERR_VALUE, "bad key width %d", bits);
  const int kRsTile = words == 1 ? RsCfg<1>::kTile : RsCfg<2>::kTile;
  const int64_t tiles = (M + kRsTile - 1) / kRsTile;
  char *p = static_cast<char *>(scratch);
  uint64_t *kalt = reinterpret_cast<uint64_t *>(p);
  p += rs_align((size_t)M * 8 * words);
  uint64_t *valt = reinterpret_cast<uint64_t *>(p);
  p += rs_align((size_t)M * 8);
  uint32_t *hist = reinterpret_cast<uint32_t *>(p);
  uint32_t *offsets = hist + kRsMaxPasses * kRsBins;
  p += rs_align((size_t)kRsMaxPasses * kRsBins * 4 * 2);
  uint32_t *status = reinterpret_cast<uint32_t *>(p);
  p += rs_align((size_t)tiles * kRsBins * 4);
  uint32_t *counters = reinterpret_cast<uint32_t *>(p);

  ALTO_CUDA(cudaMemsetAsync(hist, 0, (size_t)passes * kRsBins * 4, st));
  ALTO_CUDA(cudaMemsetAsync(counters, 0, kRsMaxPasses * 4, st));
  int hblocks = num_sms() * 4;
  const int64_t need = (M + kRsThreads - 1) / kRsThreads;
  if (need < hblocks) hblocks = (int)need;
  if (words == 1)
    rs_hist_kernel<1><<<hblocks, kRsThreads, 0, st>>>(static_cast<const uint64_t *>(keys), M, passes, hist);
  else
    rs_hist_kernel<2><<<hblocks, kRsThreads, 0, st>>>(static_cast<const uint64_t *>(keys), M, passes, hist);
  ALTO_LAUNCH_CHECK("rs_hist_kernel");
  rs_scan_kernel<<<passes, kRsBins, 0, st>>>(hist, offsets);
  ALTO_LAUNCH_CHECK("rs_scan_kernel");

  uint64_t *kin = static_cast<uint64_t *>(keys), *vin = static_cast<uint64_t *>(vals);
  uint64_t *kout = kalt, *vout = valt;
  const int smem = words == 1 ? RsSmem<1>::kBytes : RsSmem<2>::kBytes;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(rs_pass_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, RsSmem<1>::kBytes);
    cudaFuncSetAttribute(rs_pass_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, RsSmem<2>::kBytes);
    attr = true;
  }
  for (int pass = 0; pass < passes; ++pass) {
    ALTO_CUDA(cudaMemsetAsync(status, 0, (size_t)tiles * kRsBins * 4, st));
    if (words == 1)
      rs_pass_kernel<1><<<(int)tiles, kRsThreads, smem, st>>>(kin, vin, kout, vout, M, 8 * pass,
                                                               offsets + pass * kRsBins, status, counters + pass);
    else
      rs_pass_kernel<2><<<(int)tiles, kRsThreads, smem, st>>>(kin, vin, kout, vout, M, 8 * pass,
                                                               offsets + pass * kRsBins, status, counters + pass);
    ALTO_LAUNCH_CHECK("rs_pass_kernel");
    uint64_t *t = kin;
    kin = kout;
    kout = t;
    t = vin;
    vin = vout;
    vout = t;
  }
  if (kin != keys) {
    ALTO_CUDA(cudaMemcpyAsync(keys, kin, (size_t)M * 8 * words, cudaMemcpyDeviceToDevice, st));
    ALTO_CUDA(cudaMemcpyAsync(vals, vin, (size_t)M * 8, cudaMemcpyDeviceToDevice, st));
  }
  return ALTO_OK;
}

}  // namespace alto
