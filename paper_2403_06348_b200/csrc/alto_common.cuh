// Shared device helpers for the B200 ALTO kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "../../include/alto_b200.h"

namespace alto {

constexpr int kNumSMsB200 = 148;

// ---------------------------------------------------------------------------
// error plumbing (thread-local last error, status codes from alto_b200.h)

void set_error(const char *fmt, ...);
int cuda_status(cudaError_t e, const char *what);

#define ALTO_CUDA(call)                                              \
  do {                                                               \
    cudaError_t _e = (call);                                         \
    if (_e != cudaSuccess) return ::alto::cuda_status(_e, #call);    \
  } while (0)

#define ALTO_LAUNCH_CHECK(what)                                      \
  do {                                                               \
    cudaError_t _e = cudaGetLastError();                             \
    if (_e != cudaSuccess) return ::alto::cuda_status(_e, what);     \
  } while (0)

#define ALTO_REQUIRE(cond, code, ...)       \
  do {                                      \
    if (!(cond)) {                          \
      ::alto::set_error(__VA_ARGS__);       \
      return (code);                        \
    }                                       \
  } while (0)

int num_sms();
// Persistent per-thread scratch for small device flags and their pinned host
// mirror (kFlagBytes each): allocated once, never freed per call, so small
// synchronising entry points do not pay for allocation or pool trimming.
constexpr size_t kFlagBytes = 256;
int flag_scratch(void **dev, void **host);
int check_layout(const alto_layout_t *L);
int check_factors(const alto_layout_t *L, const alto_factors_t *F);
// stable LSD radix sort of (key, 8-byte payload) pairs (radix_sort.cu)
size_t radix_sort_scratch(int64_t M, int words);
// csrc/encode.cu: sort keys + stable order of a mode / fiber / blocked view
int view_sort(const alto_layout_t *host_layout, const void *keys, int64_t M, int32_t mode, int32_t second,
              int32_t bmode, int32_t bshift, int64_t *perm, void *scratch, size_t scratch_bytes, cudaStream_t st,
              uint64_t **sorted, int *second_bits);
int radix_sort_pairs(int words, int total_bits, void *keys, void *vals, int64_t M, void *scratch,
                     size_t scratch_bytes, cudaStream_t st);

// ---------------------------------------------------------------------------
// Layout tables as a kernel parameter. The table is read with warp-uniform
// indices, so it stays in the constant bank (passed as __grid_constant__).

struct Layout {
  int32_t nmodes;
  int32_t words;  // 1 or 2
  int32_t total_bits;
  int32_t nspans;
  int64_t dims[ALTO_MAX_MODES];
  int32_t span_off[ALTO_MAX_MODES + 1];
  uint8_t src[ALTO_MAX_SPANS];
  uint8_t bit[ALTO_MAX_SPANS];
  uint8_t len[ALTO_MAX_SPANS];
  uint8_t word[ALTO_MAX_SPANS];
  // Bit-compress program per mode and key word (Hacker's Delight 7-4):
  // cm[n][w][0] selects mode n's bits in word w, cm[n][w][1..6] are the
  // per-stage move masks. cshift[n] = popcount(cm[n][0][0]).
  uint64_t cm[ALTO_MAX_MODES][2][7];
  uint8_t cshift[ALTO_MAX_MODES];
};

inline void compress_masks(uint64_t m, uint64_t out[7]) {
  out[0] = m;
  uint64_t mk = ~m << 1;
  for (int i = 0; i < 6; ++i) {
    uint64_t mp = mk ^ (mk << 1);
    mp ^= mp << 2;
    mp ^= mp << 4;
    mp ^= mp << 8;
    mp ^= mp << 16;
    mp ^= mp << 32;
    const uint64_t mv = mp & m;
    m = (m ^ mv) | (mv >> (1 << i));
    mk &= ~mp;
    out[i + 1] = mv;
  }
}

inline Layout to_device_layout(const alto_layout_t *L) {
  Layout d;
  d.nmodes = L->nmodes;
  d.words = L->word_bits == 128 ? 2 : 1;
  d.total_bits = L->total_bits;
  d.nspans = L->nspans;
  for (int n = 0; n < ALTO_MAX_MODES; ++n) d.dims[n] = n < L->nmodes ? L->dims[n] : 1;
  for (int n = 0; n <= ALTO_MAX_MODES; ++n)
    d.span_off[n] = n <= L->nmodes ? L->span_off[n] : L->span_off[L->nmodes];
  for (int s = 0; s < ALTO_MAX_SPANS; ++s) {
    d.src[s] = L->span_src[s];
    d.bit[s] = L->span_bit[s];
    d.len[s] = L->span_len[s];
    d.word[s] = L->span_word[s];
  }
  for (int n = 0; n < ALTO_MAX_MODES; ++n) {
    uint64_t m[2] = {0, 0};
    if (n < L->nmodes) {
      for (int s = L->span_off[n]; s < L->span_off[n + 1]; ++s) {
        const uint64_t run = L->span_len[s] >= 64 ? ~0ull : ((1ull << L->span_len[s]) - 1ull);
        m[L->span_word[s] & 1] |= run << L->span_bit[s];
      }
    }
    compress_masks(m[0], d.cm[n][0]);
    compress_masks(m[1], d.cm[n][1]);
    d.cshift[n] = (uint8_t)__builtin_popcountll(m[0]);
  }
  return d;
}

struct Key {
  uint64_t w0, w1;
};

template <int KW>
__device__ __forceinline__ Key load_key(const uint64_t *__restrict__ keys, int64_t x) {
  Key k;
  if constexpr (KW == 1) {
    k.w0 = __ldg(keys + x);
    k.w1 = 0;
  } else {
    const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2 *>(keys) + x);
    k.w0 = v.x;
    k.w1 = v.y;
  }
  return k;
}

// streaming (read-once) loads: evict-first so the factor rows keep L1/L2
// L2 eviction-priority policies (createpolicy; the compiler hoists them)
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint64_t ld_stream_u64(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_stream_f64(const double *p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ ulonglong2 ld_stream_u64x2(const ulonglong2 *p) {
  ulonglong2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0, %1}, [%2];"
               : "=l"(v.x), "=l"(v.y) : "l"(p));
  return v;
}

template <int KW>
__device__ __forceinline__ Key load_key_stream(const uint64_t *__restrict__ keys, int64_t x) {
  Key k;
  if constexpr (KW == 1) {
    k.w0 = ld_stream_u64(keys + x);
    k.w1 = 0;
  } else {
    const ulonglong2 v = ld_stream_u64x2(reinterpret_cast<const ulonglong2 *>(keys) + x);
    k.w0 = v.x;
    k.w1 = v.y;
  }
  return k;
}

// Decode one mode's coordinate from a key (bit scatter over the span table).
__device__ __forceinline__ uint64_t decode_mode(const Layout &L, int n, const Key &k) {
  uint64_t acc = 0;
  const int s1 = L.span_off[n + 1];
  for (int s = L.span_off[n]; s < s1; ++s) {
    const uint64_t w = L.word[s] ? k.w1 : k.w0;
    const uint64_t m = (1ull << L.len[s]) - 1ull;
    acc |= ((w >> L.bit[s]) & m) << L.src[s];
  }
  return acc;
}

__device__ __forceinline__ uint64_t compress64(uint64_t x, const uint64_t (&mv)[7]) {
  x &= mv[0];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const uint64_t t = x & mv[i + 1];
    x = (x ^ t) | (t >> (1 << i));
  }
  return x;
}

// Inverse of compress64 (Hacker's Delight 7-5 "expand"): deposit the low
// popcount(mask) bits of x at the mask's bit positions, same move masks.
__device__ __forceinline__ uint64_t expand64(uint64_t x, const uint64_t (&mv)[7]) {
#pragma unroll
  for (int i = 5; i >= 0; --i) {
    const uint64_t t = x << (1 << i);
    x = (x & ~mv[i + 1]) | (t & mv[i + 1]);
  }
  return x & mv[0];
}

// Branch-free encode of mode n's coordinate c into the key (span-free).
template <int KW>
__device__ __forceinline__ void encode_fast(const Layout &L, int n, uint64_t c, Key &k) {
  const int cs = L.cshift[n];
  k.w0 |= expand64(cs >= 64 ? c : (c & ((1ull << cs) - 1ull)), L.cm[n][0]);
  if constexpr (KW == 2) k.w1 |= expand64(cs >= 64 ? 0ull : (c >> cs), L.cm[n][1]);
}

// Branch-free decode of mode n (span-free; ~38 integer ops per key word).
template <int KW>
__device__ __forceinline__ uint64_t decode_fast(const Layout &L, int n, const Key &k) {
  uint64_t c = compress64(k.w0, L.cm[n][0]);
  if constexpr (KW == 2) c |= compress64(k.w1, L.cm[n][1]) << L.cshift[n];
  return c;
}

// Encode: OR one coordinate's bits into the key words.
__device__ __forceinline__ void encode_mode(const Layout &L, int n, uint64_t c, Key &k) {
  const int s1 = L.span_off[n + 1];
  for (int s = L.span_off[n]; s < s1; ++s) {
    const uint64_t m = (1ull << L.len[s]) - 1ull;
    const uint64_t part = ((c >> L.src[s]) & m) << L.bit[s];
    if (L.word[s]) k.w1 |= part; else k.w0 |= part;
  }
}

struct Factors {
  const double *ptr[ALTO_MAX_MODES];
  int64_t ld[ALTO_MAX_MODES];
  int32_t nmodes;
  int32_t rank;
};

inline Factors to_device_factors(const alto_factors_t *F) {
  Factors f;
  for (int n = 0; n < ALTO_MAX_MODES; ++n) {
    f.ptr[n] = n < F->nmodes ? F->ptr[n] : nullptr;
    f.ld[n] = n < F->nmodes ? F->ld[n] : 0;
  }
  f.nmodes = F->nmodes;
  f.rank = F->rank;
  return f;
}

__device__ __forceinline__ void red_add_f64(double *p, double v) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

template <typename T>
__device__ __forceinline__ T shfl(T v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace alto
