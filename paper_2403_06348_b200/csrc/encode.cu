// ALTO encoder on sm_100a: linearise (bit gather), delinearise, radix sort of
// (key, value) pairs, COO canonicalisation, segment partitioning and the
// mode-ordered view. Reference stages cited per entry point in alto_b200.h.

#include <stdarg.h>
#include <string.h>

#include "alto_common.cuh"

namespace alto {

static thread_local std::string g_last_error;

void set_error(const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

int cuda_status(cudaError_t e, const char *what) {
  set_error("CUDA error in %s: %s", what, cudaGetErrorString(e));
  return ALTO_ERR_CUDA;
}

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
      sms = kNumSMsB200;
  }
  return sms;
}

int flag_scratch(void **dev, void **host) {
  static thread_local void *d = nullptr;
  static thread_local void *h = nullptr;
  static thread_local int device = -1;
  int cur = 0;
  ALTO_CUDA(cudaGetDevice(&cur));
  if (d == nullptr || device != cur) {
    ALTO_CUDA(cudaMalloc(&d, kFlagBytes));
    ALTO_CUDA(cudaMallocHost(&h, kFlagBytes));
    device = cur;
  }
  *dev = d;
  *host = h;
  return ALTO_OK;
}

int check_layout(const alto_layout_t *L) {
  ALTO_REQUIRE(L != nullptr, ALTO_ERR_VALUE, "null layout");
  ALTO_REQUIRE(L->nmodes >= 1 && L->nmodes <= ALTO_MAX_MODES, ALTO_ERR_UNSUPPORTED,
               "device kernels support 1..%d modes, got %d", ALTO_MAX_MODES, L->nmodes);
  ALTO_REQUIRE(L->word_bits == 64 || L->word_bits == 128, ALTO_ERR_VALUE, "word_bits must be 64 or 128");
  ALTO_REQUIRE(L->nspans >= 0 && L->nspans <= ALTO_MAX_SPANS, ALTO_ERR_UNSUPPORTED,
               "layout has %d spans; device limit is %d", L->nspans, ALTO_MAX_SPANS);
  ALTO_REQUIRE(L->span_off[0] == 0 && L->span_off[L->nmodes] == L->nspans, ALTO_ERR_VALUE,
               "inconsistent span table");
  return ALTO_OK;
}

int check_factors(const alto_layout_t *L, const alto_factors_t *F) {
  ALTO_REQUIRE(F != nullptr, ALTO_ERR_VALUE, "null factors");
  ALTO_REQUIRE(F->nmodes == L->nmodes, ALTO_ERR_VALUE, "expected %d factor matrices, got %d",
               L->nmodes, F->nmodes);
  ALTO_REQUIRE(F->rank >= 1, ALTO_ERR_VALUE, "rank must be positive");
  for (int n = 0; n < F->nmodes; ++n) {
    ALTO_REQUIRE(F->ld[n] >= F->rank, ALTO_ERR_VALUE, "factor %d row stride < rank", n);
  }
  return ALTO_OK;
}

// ---------------------------------------------------------------------------

static int grid_for(int64_t work, int block) {
  int64_t g = ceil_div(work, block);
  int64_t cap = (int64_t)num_sms() * 8;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

// NM > 0: mode count known at compile time (bit-deposit encode, unrolled);
// NM == 0: any mode count (same arithmetic, runtime loop)
template <int KW, int NM>
__global__ void encode_kernel(const __grid_constant__ Layout L, const int64_t *__restrict__ coords,
                              int64_t M, uint64_t *__restrict__ keys,
                              unsigned long long *__restrict__ bad_row) {
  const int N = NM > 0 ? NM : L.nmodes;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < M;
       x += (int64_t)gridDim.x * blockDim.x) {
    Key k{0, 0};
    bool bad = false;
#pragma unroll
    for (int n = 0; n < (NM > 0 ? NM : ALTO_MAX_MODES); ++n) {
      if (NM == 0 && n >= N) break;
      const int64_t c = coords[x * N + n];
      if (c < 0 || c >= L.dims[n]) bad = true;
      encode_fast<KW>(L, n, (uint64_t)c, k);
    }
    if (bad) atomicMin(bad_row, (unsigned long long)x);
    if constexpr (KW == 1) {
      keys[x] = k.w0;
    } else {
      reinterpret_cast<ulonglong2 *>(keys)[x] = make_ulonglong2(k.w0, k.w1);
    }
  }
}

template <int KW>
__global__ void decode_kernel(const __grid_constant__ Layout L, const uint64_t *__restrict__ keys,
                              int64_t M, int64_t *__restrict__ coords) {
  const int N = L.nmodes;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < M;
       x += (int64_t)gridDim.x * blockDim.x) {
    const Key k = load_key<KW>(keys, x);
    for (int n = 0; n < N; ++n) coords[x * N + n] = (int64_t)decode_mode(L, n, k);
  }
}

__global__ void validate_kernel(const int64_t *__restrict__ coords, const double *__restrict__ vals,
                                int64_t M, int N, const __grid_constant__ Layout L,
                                unsigned long long *__restrict__ flags) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < M;
       x += (int64_t)gridDim.x * blockDim.x) {
    bool bad = false;
    for (int n = 0; n < N; ++n) {
      const int64_t c = coords[x * N + n];
      bad |= (c < 0) | (c >= L.dims[n]);
    }
    if (bad) atomicMin(flags, (unsigned long long)x);
    if (!isfinite(vals[x])) atomicMin(flags + 1, (unsigned long long)x);
  }
}

// All sorts (encoder, canonicalisation, mode/fiber views) go through the
// hand-written stable LSD radix sort in radix_sort.cu.
template <typename V>
static int sort_pairs_impl(int words, int total_bits, void *keys, V *vals, int64_t M,
                           void *scratch, size_t scratch_bytes, cudaStream_t st) {
  static_assert(sizeof(V) == 8, "8-byte payloads");
  return radix_sort_pairs(words, total_bits, keys, vals, M, scratch, scratch_bytes, st);
}

// ---- stable stream compaction (canonicalisation: keep the duplicate-run
// heads whose sum is nonzero) -------------------------------------------
// Tiles of kCompactTile flags: per-tile counts, one exclusive scan of the
// tile counts, then every tile recounts its flags with a block scan and
// writes its kept keys / values in input order.
constexpr int kCompactThreads = 256;
constexpr int kCompactPer = 16;
constexpr int64_t kCompactTile = (int64_t)kCompactThreads * kCompactPer;

static int64_t compact_tiles(int64_t M) { return (M + kCompactTile - 1) / kCompactTile; }

__global__ void __launch_bounds__(kCompactThreads) compact_count_kernel(const unsigned char *__restrict__ keep,
                                                                       int64_t M, int64_t *__restrict__ counts) {
  const int64_t t0 = blockIdx.x * kCompactTile;
  int c = 0;
  for (int i = threadIdx.x; i < kCompactTile; i += kCompactThreads) {
    const int64_t x = t0 + i;
    c += (x < M && keep[x]) ? 1 : 0;
  }
  c = __reduce_add_sync(0xffffffffu, c);
  __shared__ int w[kCompactThreads / 32];
  if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int i = 0; i < kCompactThreads / 32; ++i) t += w[i];
    counts[blockIdx.x] = t;
  }
}

// exclusive scan of n tile counts in place; total -> out_total (one block)
__global__ void __launch_bounds__(1024) compact_scan_kernel(int64_t *__restrict__ counts, int64_t n,
                                                           int64_t *__restrict__ out_total) {
  __shared__ int64_t part[1024];
  const int t = threadIdx.x, T = blockDim.x;
  const int64_t per = (n + T - 1) / T;
  const int64_t b = t * per, e = b + per < n ? b + per : n;
  int64_t sum = 0;
  for (int64_t i = b; i < e; ++i) sum += counts[i];
  part[t] = sum;
  __syncthreads();
  if (t == 0) {
    int64_t acc = 0;
    for (int i = 0; i < T; ++i) {
      const int64_t v = part[i];
      part[i] = acc;
      acc += v;
    }
    *out_total = acc;
  }
  __syncthreads();
  int64_t acc = part[t];
  for (int64_t i = b; i < e; ++i) {
    const int64_t v = counts[i];
    counts[i] = acc;
    acc += v;
  }
}

template <int KW>
__global__ void __launch_bounds__(kCompactThreads) compact_scatter_kernel(
    const uint64_t *__restrict__ keys, const double *__restrict__ vals, const unsigned char *__restrict__ keep,
    int64_t M, const int64_t *__restrict__ tile_off, uint64_t *__restrict__ keys_out,
    double *__restrict__ vals_out) {
  // each thread owns kCompactPer consecutive flags of the tile (stable order)
  const int64_t x0 = blockIdx.x * kCompactTile + (int64_t)threadIdx.x * kCompactPer;
  int c = 0;
#pragma unroll
  for (int i = 0; i < kCompactPer; ++i) c += (x0 + i < M && keep[x0 + i]) ? 1 : 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int inc = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  __shared__ int w[kCompactThreads / 32];
  if (lane == 31) w[warp] = inc;
  __syncthreads();
  int before = 0;
  for (int i = 0; i < warp; ++i) before += w[i];
  int64_t pos = tile_off[blockIdx.x] + before + inc - c;
#pragma unroll
  for (int i = 0; i < kCompactPer; ++i) {
    const int64_t x = x0 + i;
    if (x < M && keep[x]) {
      if (KW == 1) {
        keys_out[pos] = keys[x];
      } else {
        keys_out[2 * pos] = keys[2 * x];
        keys_out[2 * pos + 1] = keys[2 * x + 1];
      }
      vals_out[pos] = vals[x];
      ++pos;
    }
  }
}

static size_t sort_scratch(int64_t M, int words) {
  auto align = [](size_t b) { return (b + 255) & ~size_t(255); };
  // canonicalisation carves [idx | sums | keep | nsel] first; the rest holds
  // the sort's buffers, later the compaction's staging + temp
  size_t region = radix_sort_scratch(M, words);
  const size_t compact = align((size_t)M * 16) + align((size_t)compact_tiles(M) * 8) + 256;
  if (compact > region) region = compact;
  return align((size_t)M * 8) * 2 + align((size_t)M + 16) + 256 + region + 4096;
}

// ---- canonicalisation ------------------------------------------------------

template <int KW>
__device__ __forceinline__ bool key_eq(const uint64_t *keys, int64_t a, int64_t b) {
  if constexpr (KW == 1) return keys[a] == keys[b];
  else return keys[2 * a] == keys[2 * b] && keys[2 * a + 1] == keys[2 * b + 1];
}

// number of sorted keys strictly below each query key (binary search; keys
// in ascending numeric order, 128-bit keys compare hi word first)
template <int KW>
__global__ void count_less_kernel(const uint64_t *__restrict__ keys, int64_t M, const uint64_t *__restrict__ q,
                                  int nq, int64_t *__restrict__ counts) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nq) return;
  const uint64_t qlo = KW == 1 ? q[i] : q[2 * i], qhi = KW == 1 ? 0 : q[2 * i + 1];
  int64_t lo = 0, hi = M;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    bool less;
    if constexpr (KW == 1) {
      less = keys[mid] < qlo;
    } else {
      const uint64_t khi = keys[2 * mid + 1], klo = keys[2 * mid];
      less = khi < qhi || (khi == qhi && klo < qlo);
    }
    if (less) lo = mid + 1;
    else hi = mid;
  }
  counts[i] = lo;
}

// Heads of equal-key runs sum their members sequentially in input order
// (stable sort keeps input order within a run), matching np.add.at's
// summed[u] = ((0 + v_a) + v_b) + ... (pkg/src/alto/tensor.py:120-123).
template <int KW>
__global__ void merge_runs_kernel(const uint64_t *__restrict__ keys, const int64_t *__restrict__ idx,
                                  const double *__restrict__ vals_in, int64_t M,
                                  double *__restrict__ sums, unsigned char *__restrict__ keep) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < M;
       x += (int64_t)gridDim.x * blockDim.x) {
    const bool head = (x == 0) || !key_eq<KW>(keys, x, x - 1);
    if (!head) {
      keep[x] = 0;
      continue;
    }
    // the adds are sequential by contract; the loads are not: a batch's
    // run-membership tests, index loads and value gathers are issued
    // together (a long run of duplicates paid two dependent L2 / DRAM
    // latencies per member: 0.95 s for the hottest run of the c2 generator's
    // draws, profiles/r02_build_fused.txt)
    constexpr int B = 16;
    double s = 0.0;
    int64_t j = x;
    bool more = true;
    if (x + 1 >= M || !key_eq<KW>(keys, x + 1, x)) {
      // a run of one (canonical input: every key): no batch
      s = __dadd_rn(s, vals_in[idx[x]]);
      more = false;
    }
    while (more) {
      bool in[B];
      double v[B];
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const int64_t jj = j + b;
        in[b] = jj == x || (jj < M && key_eq<KW>(keys, jj, x));
      }
#pragma unroll
      for (int b = 0; b < B; ++b) v[b] = in[b] ? vals_in[idx[j + b]] : 0.0;
#pragma unroll
      for (int b = 0; b < B; ++b) {
        // equal keys are contiguous: the first miss ends the run
        more = more && in[b];
        if (more) s = __dadd_rn(s, v[b]);
      }
      j += B;
    }
    sums[x] = s;
    keep[x] = (s != 0.0);
  }
}

__global__ void iota_kernel(int64_t *p, int64_t M) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < M;
       x += (int64_t)gridDim.x * blockDim.x)
    p[x] = x;
}

// ---- partition -----------------------------------------------------------

__device__ __forceinline__ int64_t balanced_segment_of(int64_t x, int64_t M, int64_t L) {
  const int64_t base = M / L, extra = M % L;
  const int64_t cut = extra * (base + 1);
  return x < cut ? x / (base + 1) : extra + (x - cut) / base;
}

__global__ void bounds_kernel(int64_t M, int L, int64_t *bounds) {
  const int64_t base = M / L, extra = M % L;
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l <= L;
       l += (int64_t)gridDim.x * blockDim.x)
    bounds[l] = l * base + (l < extra ? l : extra);
}

__global__ void fill_u64_kernel(unsigned long long *p, int64_t n, unsigned long long v) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x)
    p[x] = v;
}

template <int KW>
__global__ void intervals_kernel(const __grid_constant__ Layout L, const uint64_t *__restrict__ keys,
                                 int64_t M, int nseg, unsigned long long *__restrict__ lo,
                                 unsigned long long *__restrict__ hi) {
  const int N = L.nmodes;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // iterate in warp-aligned steps so every lane of a warp reaches the shuffles
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) - lane; base < M;
       base += stride) {
    const int64_t x = base + lane;
    const bool valid = x < M;
    const int64_t seg = valid ? balanced_segment_of(x, M, nseg) : -1;
    const int64_t seg0 = __shfl_sync(0xffffffffu, seg, 0);
    const bool uniform = __all_sync(0xffffffffu, !valid || seg == seg0);
    Key k{0, 0};
    if (valid) k = load_key<KW>(keys, x);
    for (int n = 0; n < N; ++n) {
      const unsigned long long c = valid ? decode_mode(L, n, k) : 0ull;
      if (uniform) {
        unsigned long long mn = valid ? c : ~0ull, mx = valid ? c : 0ull;
        for (int o = 16; o; o >>= 1) {
          mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
          mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (lane == 0) {
          atomicMin(lo + seg0 * N + n, mn);
          atomicMax(hi + seg0 * N + n, mx);
        }
      } else if (valid) {
        atomicMin(lo + seg * N + n, c);
        atomicMax(hi + seg * N + n, c);
      }
    }
  }
}

template <int KW>
__global__ void row_span_kernel(const __grid_constant__ Layout L, const uint64_t *__restrict__ keys,
                                int64_t M, int mode, int nseg, int *__restrict__ rmin,
                                int *__restrict__ rmax) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < M;
       x += (int64_t)gridDim.x * blockDim.x) {
    const Key k = load_key<KW>(keys, x);
    const uint64_t r = decode_mode(L, mode, k);
    const int s = (int)balanced_segment_of(x, M, nseg);
    atomicMin(rmin + r, s);
    atomicMax(rmax + r, s);
  }
}

__global__ void fill_i32_kernel(int *p, int64_t n, int v) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x)
    p[x] = v;
}

template <int KW>
__global__ void mode_coord_kernel(const __grid_constant__ Layout L, const uint64_t *__restrict__ keys,
                                  int64_t M, int mode, int second, int sbits, int bmode, int bshift,
                                  int hbits, uint64_t *__restrict__ rows, int64_t *__restrict__ idx) {
  // sort key: [block of bmode coordinate | mode coordinate | second coordinate]
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < M;
       x += (int64_t)gridDim.x * blockDim.x) {
    // branch-free bit-compress decode (the span loop measured 1.9 ms per
    // c2 view, this 0.4: profiles/r02_build_fused.txt)
    const Key k = load_key<KW>(keys, x);
    uint64_t r = decode_fast<KW>(L, mode, k);
    if (second >= 0) r = (r << sbits) | decode_fast<KW>(L, second, k);
    if (bmode >= 0) r |= (decode_fast<KW>(L, bmode, k) >> bshift) << hbits;
    rows[x] = r;
    idx[x] = x;
  }
}

template <int KW>
__global__ void gather_pairs_kernel(const int64_t *__restrict__ perm, const uint64_t *__restrict__ keys,
                                    const double *__restrict__ vals, int64_t M,
                                    uint64_t *__restrict__ out_keys, double *__restrict__ out_vals) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < M;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = perm[x];
    if constexpr (KW == 1) {
      out_keys[x] = keys[p];
    } else {
      reinterpret_cast<ulonglong2 *>(out_keys)[x] = reinterpret_cast<const ulonglong2 *>(keys)[p];
    }
    out_vals[x] = vals[p];
  }
}

}  // namespace alto

using namespace alto;

extern "C" {

int alto_abi_version(void) { return 1; }

const char *alto_last_error(void) { return g_last_error.c_str(); }

int alto_device_sm_count(int32_t *host_sms) {
  *host_sms = num_sms();
  return ALTO_OK;
}

int alto_encode(const alto_layout_t *host_layout, const int64_t *coords, int64_t M, void *keys,
                int64_t *host_bad_row, void *stream) {
  int rc = check_layout(host_layout);
  if (rc) return rc;
  *host_bad_row = -1;
  if (M <= 0) return ALTO_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Layout L = to_device_layout(host_layout);
  void *dflag = nullptr, *hflag = nullptr;
  rc = flag_scratch(&dflag, &hflag);
  if (rc) return rc;
  unsigned long long *flag = static_cast<unsigned long long *>(dflag);
  fill_u64_kernel<<<1, 32, 0, st>>>(flag, 1, ~0ull);
  const int g = grid_for(M, 256);
  uint64_t *k = static_cast<uint64_t *>(keys);
#define ALTO_ENC(KW, NM) encode_kernel<KW, NM><<<g, 256, 0, st>>>(L, coords, M, k, flag)
  if (L.words == 1) {
    switch (L.nmodes) {
      case 2: ALTO_ENC(1, 2); break;
      case 3: ALTO_ENC(1, 3); break;
      case 4: ALTO_ENC(1, 4); break;
      case 5: ALTO_ENC(1, 5); break;
      default: ALTO_ENC(1, 0);
    }
  } else {
    switch (L.nmodes) {
      case 3: ALTO_ENC(2, 3); break;
      case 4: ALTO_ENC(2, 4); break;
      case 5: ALTO_ENC(2, 5); break;
      default: ALTO_ENC(2, 0);
    }
  }
#undef ALTO_ENC
  ALTO_LAUNCH_CHECK("encode_kernel");
  ALTO_CUDA(cudaMemcpyAsync(hflag, flag, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  ALTO_CUDA(cudaStreamSynchronize(st));
  const unsigned long long h = *static_cast<unsigned long long *>(hflag);
  if (h != ~0ull) {
    *host_bad_row = (int64_t)h;
    set_error("coordinate out of range in row %lld", (long long)h);
    return ALTO_ERR_INDEX;
  }
  return ALTO_OK;
}

int alto_decode(const alto_layout_t *host_layout, const void *keys, int64_t M, int64_t *coords,
                void *stream) {
  int rc = check_layout(host_layout);
  if (rc) return rc;
  if (M <= 0) return ALTO_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Layout L = to_device_layout(host_layout);
  const int g = grid_for(M, 256);
  if (L.words == 1)
    decode_kernel<1><<<g, 256, 0, st>>>(L, static_cast<const uint64_t *>(keys), M, coords);
  else
    decode_kernel<2><<<g, 256, 0, st>>>(L, static_cast<const uint64_t *>(keys), M, coords);
  ALTO_LAUNCH_CHECK("decode_kernel");
  return ALTO_OK;
}

int alto_validate_coo(const int64_t *coords, const double *vals, int64_t M, int32_t N,
                      const int64_t *host_dims, int64_t *host_flags, void *stream) {
  host_flags[0] = host_flags[1] = -1;
  if (M <= 0) return ALTO_OK;
  ALTO_REQUIRE(N >= 1 && N <= ALTO_MAX_MODES, ALTO_ERR_UNSUPPORTED, "bad mode count %d", N);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  alto_layout_t tmp;
  memset(&tmp, 0, sizeof tmp);
  tmp.nmodes = N;
  tmp.word_bits = 64;
  for (int n = 0; n < N; ++n) tmp.dims[n] = host_dims[n];
  const Layout L = to_device_layout(&tmp);
  void *dflag = nullptr, *hflag = nullptr;
  int rc = flag_scratch(&dflag, &hflag);
  if (rc) return rc;
  unsigned long long *flags = static_cast<unsigned long long *>(dflag);
  fill_u64_kernel<<<1, 32, 0, st>>>(flags, 2, ~0ull);
  validate_kernel<<<grid_for(M, 256), 256, 0, st>>>(coords, vals, M, N, L, flags);
  ALTO_LAUNCH_CHECK("validate_kernel");
  ALTO_CUDA(cudaMemcpyAsync(hflag, flags, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  ALTO_CUDA(cudaStreamSynchronize(st));
  const unsigned long long *h = static_cast<const unsigned long long *>(hflag);
  host_flags[0] = h[0] == ~0ull ? -1 : (int64_t)h[0];
  host_flags[1] = h[1] == ~0ull ? -1 : (int64_t)h[1];
  return ALTO_OK;
}

int alto_sort_scratch_bytes(int64_t M, int32_t word_bits, size_t *host_bytes) {
  *host_bytes = sort_scratch(M < 1 ? 1 : M, word_bits == 128 ? 2 : 1);
  return ALTO_OK;
}

int alto_sort_pairs(const alto_layout_t *host_layout, void *keys, double *vals, int64_t M,
                    void *scratch, size_t scratch_bytes, void *stream) {
  int rc = check_layout(host_layout);
  if (rc) return rc;
  if (M <= 1) return ALTO_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return sort_pairs_impl<double>(host_layout->word_bits == 128 ? 2 : 1, host_layout->total_bits,
                                 keys, vals, M, scratch, scratch_bytes, st);
}

int alto_canonicalize(const alto_layout_t *host_lex_layout, void *keys, double *vals, int64_t M,
                      void *scratch, size_t scratch_bytes, int64_t *host_M_out, void *stream) {
  int rc = check_layout(host_lex_layout);
  if (rc) return rc;
  *host_M_out = 0;
  if (M <= 0) return ALTO_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int words = host_lex_layout->word_bits == 128 ? 2 : 1;
  auto align = [](size_t b) { return (b + 255) & ~size_t(255); };
  // scratch: [idx | sums | keep | keys_out | cub sort scratch...]
  char *base = static_cast<char *>(scratch);
  int64_t *idx = reinterpret_cast<int64_t *>(base);
  size_t off = align((size_t)M * 8);
  double *sums = reinterpret_cast<double *>(base + off);
  off += align((size_t)M * 8);
  unsigned char *keep = reinterpret_cast<unsigned char *>(base + off);
  off += align((size_t)M + 16);
  int64_t *nsel = reinterpret_cast<int64_t *>(base + off);
  off += 256;
  ALTO_REQUIRE(scratch_bytes > off, ALTO_ERR_VALUE, "canonicalize scratch too small");
  const int g = grid_for(M, 256);
  iota_kernel<<<g, 256, 0, st>>>(idx, M);
  rc = sort_pairs_impl<int64_t>(words, host_lex_layout->total_bits, keys, idx, M, base + off,
                                scratch_bytes - off, st);
  if (rc) return rc;
  if (words == 1)
    merge_runs_kernel<1><<<g, 256, 0, st>>>(static_cast<uint64_t *>(keys), idx, vals, M, sums, keep);
  else
    merge_runs_kernel<2><<<g, 256, 0, st>>>(static_cast<uint64_t *>(keys), idx, vals, M, sums, keep);
  ALTO_LAUNCH_CHECK("merge_runs_kernel");
  // compact heads that survived (the sort's scratch is free again): keys
  // into staging, the sums straight into vals (the input values are consumed)
  char *temp = base + off;
  size_t temp_bytes = scratch_bytes - off;
  const int64_t tiles = compact_tiles(M);
  const size_t kbytes = align((size_t)M * 8 * words);
  ALTO_REQUIRE(temp_bytes >= kbytes + align((size_t)tiles * 8), ALTO_ERR_VALUE, "canonicalize scratch too small");
  uint64_t *kout = reinterpret_cast<uint64_t *>(temp);
  int64_t *tile_off = reinterpret_cast<int64_t *>(temp + kbytes);
  compact_count_kernel<<<(int)tiles, kCompactThreads, 0, st>>>(keep, M, tile_off);
  ALTO_LAUNCH_CHECK("compact_count_kernel");
  compact_scan_kernel<<<1, 1024, 0, st>>>(tile_off, tiles, nsel);
  ALTO_LAUNCH_CHECK("compact_scan_kernel");
  uint64_t *k = static_cast<uint64_t *>(keys);
  if (words == 1)
    compact_scatter_kernel<1><<<(int)tiles, kCompactThreads, 0, st>>>(k, sums, keep, M, tile_off, kout, vals);
  else
    compact_scatter_kernel<2><<<(int)tiles, kCompactThreads, 0, st>>>(k, sums, keep, M, tile_off, kout, vals);
  ALTO_LAUNCH_CHECK("compact_scatter_kernel");
  ALTO_CUDA(cudaMemcpyAsync(k, kout, (size_t)M * 8 * words, cudaMemcpyDeviceToDevice, st));
  int64_t h = 0;
  ALTO_CUDA(cudaMemcpyAsync(&h, nsel, sizeof h, cudaMemcpyDeviceToHost, st));
  ALTO_CUDA(cudaStreamSynchronize(st));
  *host_M_out = h;
  return ALTO_OK;
}

int alto_partition(const alto_layout_t *host_layout, const void *keys, int64_t M, int32_t L,
                   int64_t *bounds, int64_t *lo, int64_t *hi, void *stream) {
  int rc = check_layout(host_layout);
  if (rc) return rc;
  ALTO_REQUIRE(L >= 1 && L <= M, ALTO_ERR_VALUE, "need 1 <= segments <= nnz");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Layout D = to_device_layout(host_layout);
  const int N = D.nmodes;
  bounds_kernel<<<grid_for(L + 1, 256), 256, 0, st>>>(M, L, bounds);
  fill_u64_kernel<<<grid_for((int64_t)L * N, 256), 256, 0, st>>>(
      reinterpret_cast<unsigned long long *>(lo), (int64_t)L * N, ~0ull);
  fill_u64_kernel<<<grid_for((int64_t)L * N, 256), 256, 0, st>>>(
      reinterpret_cast<unsigned long long *>(hi), (int64_t)L * N, 0ull);
  const int g = grid_for(M, 256);
  if (D.words == 1)
    intervals_kernel<1><<<g, 256, 0, st>>>(D, static_cast<const uint64_t *>(keys), M, L,
                                           reinterpret_cast<unsigned long long *>(lo),
                                           reinterpret_cast<unsigned long long *>(hi));
  else
    intervals_kernel<2><<<g, 256, 0, st>>>(D, static_cast<const uint64_t *>(keys), M, L,
                                           reinterpret_cast<unsigned long long *>(lo),
                                           reinterpret_cast<unsigned long long *>(hi));
  ALTO_LAUNCH_CHECK("intervals_kernel");
  return ALTO_OK;
}

int alto_count_less(int32_t word_bits, const void *keys, int64_t M, const void *queries, int32_t nq,
                    int64_t *counts, void *stream) {
  ALTO_REQUIRE(word_bits == 64 || word_bits == 128, ALTO_ERR_VALUE, "word_bits must be 64 or 128");
  if (nq <= 0) return ALTO_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int g = (nq + 127) / 128;
  if (word_bits == 64)
    count_less_kernel<1><<<g, 128, 0, st>>>(static_cast<const uint64_t *>(keys), M,
                                            static_cast<const uint64_t *>(queries), nq, counts);
  else
    count_less_kernel<2><<<g, 128, 0, st>>>(static_cast<const uint64_t *>(keys), M,
                                            static_cast<const uint64_t *>(queries), nq, counts);
  ALTO_LAUNCH_CHECK("count_less_kernel");
  return ALTO_OK;
}

int alto_row_segment_span(const alto_layout_t *host_layout, const void *keys, int64_t M,
                          int32_t mode, const int64_t *bounds, int32_t L, int32_t *row_min,
                          int32_t *row_max, void *stream) {
  (void)bounds;
  int rc = check_layout(host_layout);
  if (rc) return rc;
  ALTO_REQUIRE(mode >= 0 && mode < host_layout->nmodes, ALTO_ERR_VALUE, "mode %d out of range", mode);
  ALTO_REQUIRE(L >= 1 && L <= M, ALTO_ERR_VALUE, "need 1 <= segments <= nnz");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Layout D = to_device_layout(host_layout);
  const int64_t I = D.dims[mode];
  fill_i32_kernel<<<grid_for(I, 256), 256, 0, st>>>(row_min, I, 0x7fffffff);
  fill_i32_kernel<<<grid_for(I, 256), 256, 0, st>>>(row_max, I, -1);
  const int g = grid_for(M, 256);
  if (D.words == 1)
    row_span_kernel<1><<<g, 256, 0, st>>>(D, static_cast<const uint64_t *>(keys), M, mode, L, row_min, row_max);
  else
    row_span_kernel<2><<<g, 256, 0, st>>>(D, static_cast<const uint64_t *>(keys), M, mode, L, row_min, row_max);
  ALTO_LAUNCH_CHECK("row_span_kernel");
  return ALTO_OK;
}

int alto_mode_view_scratch_bytes(int64_t M, size_t *host_bytes) {
  *host_bytes = sort_scratch(M < 1 ? 1 : M, 1) + (size_t)(M < 1 ? 1 : M) * 16 + 512;
  return ALTO_OK;
}

static int mode_view_impl(const alto_layout_t *host_layout, const void *keys, const double *vals,
                          int64_t M, int32_t mode, int32_t second, int64_t *perm, void *view_keys,
                          double *view_vals, void *scratch, size_t scratch_bytes, void *stream,
                          int32_t bmode = -1, int32_t bshift = 0);

int alto_mode_view(const alto_layout_t *host_layout, const void *keys, const double *vals,
                   int64_t M, int32_t mode, int64_t *perm, void *view_keys, double *view_vals,
                   void *scratch, size_t scratch_bytes, void *stream) {
  return mode_view_impl(host_layout, keys, vals, M, mode, -1, perm, view_keys, view_vals, scratch,
                        scratch_bytes, stream);
}

int alto_fiber_view(const alto_layout_t *host_layout, const void *keys, const double *vals,
                    int64_t M, int32_t mode, int32_t fiber_mode, int64_t *perm, void *view_keys,
                    double *view_vals, void *scratch, size_t scratch_bytes, void *stream) {
  ALTO_REQUIRE(fiber_mode >= 0 && fiber_mode < host_layout->nmodes && fiber_mode != mode,
               ALTO_ERR_VALUE, "fiber mode %d invalid for mode %d", fiber_mode, mode);
  return mode_view_impl(host_layout, keys, vals, M, mode, fiber_mode, perm, view_keys, view_vals,
                        scratch, scratch_bytes, stream);
}

int alto_blocked_view(const alto_layout_t *host_layout, const void *keys, const double *vals, int64_t M,
                      int32_t mode, int32_t fiber_mode, int32_t block_mode, int32_t block_shift, int64_t *perm,
                      void *view_keys, double *view_vals, void *scratch, size_t scratch_bytes, void *stream) {
  ALTO_REQUIRE(block_mode >= 0 && block_mode < host_layout->nmodes && block_mode != mode, ALTO_ERR_VALUE,
               "block mode %d invalid for mode %d", block_mode, mode);
  ALTO_REQUIRE(block_shift >= 0 && block_shift < 63, ALTO_ERR_VALUE, "bad block shift %d", block_shift);
  return mode_view_impl(host_layout, keys, vals, M, mode, fiber_mode, perm, view_keys, view_vals, scratch,
                        scratch_bytes, stream, block_mode, block_shift);
}

static int mode_view_impl(const alto_layout_t *host_layout, const void *keys, const double *vals,
                          int64_t M, int32_t mode, int32_t second, int64_t *perm, void *view_keys,
                          double *view_vals, void *scratch, size_t scratch_bytes, void *stream, int32_t bmode,
                          int32_t bshift) {
  if (M <= 0) {
    int rc = check_layout(host_layout);
    if (rc) return rc;
    ALTO_REQUIRE(mode >= 0 && mode < host_layout->nmodes, ALTO_ERR_VALUE, "mode %d out of range", mode);
    return ALTO_OK;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint64_t *rows = nullptr;
  int sbits = 0;
  int rc = alto::view_sort(host_layout, keys, M, mode, second, bmode, bshift, perm, scratch, scratch_bytes, st, &rows,
                           &sbits);
  if (rc) return rc;
  const int g = grid_for(M, 256);
  if (host_layout->word_bits == 64)
    gather_pairs_kernel<1><<<g, 256, 0, st>>>(perm, static_cast<const uint64_t *>(keys), vals, M,
                                              static_cast<uint64_t *>(view_keys), view_vals);
  else
    gather_pairs_kernel<2><<<g, 256, 0, st>>>(perm, static_cast<const uint64_t *>(keys), vals, M,
                                              static_cast<uint64_t *>(view_keys), view_vals);
  ALTO_LAUNCH_CHECK("gather_pairs_kernel");
  return ALTO_OK;
}

}  // extern "C"

namespace alto {

// Sort keys [block | mode coordinate | second-mode coordinate] of every
// nonzero and the stable order by them: `*sorted` (in `scratch`) holds the
// sorted sort keys, `perm` the source positions (the first half of every view
// build; pkg/src/alto/partition.py:185-188's stable argsort).
int view_sort(const alto_layout_t *host_layout, const void *keys, int64_t M, int32_t mode, int32_t second,
              int32_t bmode, int32_t bshift, int64_t *perm, void *scratch, size_t scratch_bytes, cudaStream_t st,
              uint64_t **sorted, int *second_bits) {
  int rc = check_layout(host_layout);
  if (rc) return rc;
  ALTO_REQUIRE(mode >= 0 && mode < host_layout->nmodes, ALTO_ERR_VALUE, "mode %d out of range", mode);
  ALTO_REQUIRE(M > 0, ALTO_ERR_VALUE, "empty tensor");
  const Layout D = to_device_layout(host_layout);
  auto align = [](size_t b) { return (b + 255) & ~size_t(255); };
  char *base = static_cast<char *>(scratch);
  uint64_t *rows = reinterpret_cast<uint64_t *>(base);
  size_t off = align((size_t)M * 8);
  ALTO_REQUIRE(scratch_bytes > off, ALTO_ERR_VALUE, "view scratch too small");
  const int g = grid_for(M, 256);
  auto nbits = [](int64_t d) {
    int b = 0;
    while (b < 63 && (1ll << b) < d) ++b;
    return b;
  };
  const int sbits = second >= 0 ? nbits(D.dims[second]) : 0;
  const int hbits = nbits(D.dims[mode]) + sbits;
  int bbits = 0;
  if (bmode >= 0) {
    bbits = nbits(D.dims[bmode]) - bshift;
    if (bbits < 0) bbits = 0;
  }
  int bits = hbits + bbits;
  ALTO_REQUIRE(bits <= 64, ALTO_ERR_UNSUPPORTED, "view sort key needs %d bits", bits);
  if (bits < 1) bits = 1;
  if (D.words == 1)
    mode_coord_kernel<1><<<g, 256, 0, st>>>(D, static_cast<const uint64_t *>(keys), M, mode, second, sbits,
                                            bbits ? bmode : -1, bshift, hbits, rows, perm);
  else
    mode_coord_kernel<2><<<g, 256, 0, st>>>(D, static_cast<const uint64_t *>(keys), M, mode, second, sbits,
                                            bbits ? bmode : -1, bshift, hbits, rows, perm);
  ALTO_LAUNCH_CHECK("mode_coord_kernel");
  rc = sort_pairs_impl<int64_t>(1, bits, rows, perm, M, base + off, scratch_bytes - off, st);
  if (rc) return rc;
  *sorted = rows;
  *second_bits = sbits;
  return ALTO_OK;
}

}  // namespace alto
