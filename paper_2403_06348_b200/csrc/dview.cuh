// Decoded-view kernel helpers shared by dview_kernels.cu and memo_sums.cu:
// the argument block, segment and staging constants (per-lane cp.async and
// the interleaved bulk-copy layout), the end-of-segment flush and predicated
// vector load/store.
#pragma once

#include <string.h>

#include "det.cuh"
#include "run_kernels.cuh"
#include "tma.cuh"

namespace alto {

// row stride of the SoA coordinate block: M rounded up to 8 so every row is
// 32-byte aligned for the vector stream loads (mirrored by partition.py)
__host__ __device__ inline int64_t crd_stride(int64_t M) { return (M + 7) & ~int64_t(7); }

struct DViewArgs {
  const uint32_t *rows;  // [M]
  const uint32_t *crd;   // [N-1][M] other modes, ascending
  const double *vals;    // [M]
  int64_t M;
  int64_t crd_ld;  // row stride of crd (M rounded up to 8)
  int32_t nmodes;
  int32_t mode;
  int32_t rank;
  int32_t col0;
  int64_t nseg;
  const double *fptr[ALTO_MAX_MODES];  // other modes, ascending (N-1 used)
  int64_t fld[ALTO_MAX_MODES];
  double *out;
  int64_t ldo;
  const double *scaled;
  int64_t lds;
  const double *pi;  // PRE: Khatri-Rao rows in view order (Phi), or null
  int64_t ldp;
  double eps;
  const int32_t *skip;  // device flag: return at once when set (device-driven APR loop), or null
  int32_t reduce_all;   // rows recur across the view (blocked views): reduce every run
  double *pi_il;        // Phi (OTF): also store the Khatri-Rao rows, lane-interleaved (pstream.cu), or null
  // memoised CP-ALS sweep (memo0_kernel): fiber pieces of the view
  const uint32_t *m_pbase;  // [nseg + 1] first piece of every segment
  double *m_T;              // [P][m_ldT] piece sums sum_x v_x A_k[k_x], piece order
  int64_t m_ldT;
  DetEdges det;  // deterministic mode: edge runs parked per segment (det.cu), or det.val == null
};

// fixed 512-nonzero segments (aligned); each lane streams 4 consecutive
// nonzeros per field, so a warp-wide stream load serves 8 groups x 4G
// nonzeros
constexpr int kDvSeg = 512;

__device__ __forceinline__ uint32_t pick(const uint4 &v, int e) {
  return e == 0 ? v.x : (e == 1 ? v.y : (e == 2 ? v.z : v.w));
}

// dview3: the stream is staged in shared memory with cp.async: each lane
// copies its 4 consecutive nonzeros per field (16 B per u32 field, 32 B of
// values) S-1 chunks ahead, and the group reads a quad back with 128-bit
// broadcast LDS (group regions padded by 16 B so the groups of a warp hit
// disjoint banks: one wavefront per LDS); the registers go to gathers
// (U = 4 nonzeros per batch for MTTKRP).
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, int src_bytes) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

#ifndef DV3_QPC
#define DV3_QPC 0  // quads (4 nonzeros) per group chunk; 0: G (every lane copies one quad)
#endif
template <int G>
constexpr int dv3_quads() {
  return (DV3_QPC > 0 && DV3_QPC < G) ? DV3_QPC : G;
}

template <int NO, int G>
struct Dv3Smem {
  static constexpr int Q = dv3_quads<G>();
  static constexpr int NG = 32 / G;        // groups per warp
  static constexpr int GS = 16 * Q + 16;   // bytes per group, u32 field
  static constexpr int VS = 32 * Q + 16;   // bytes per group, values
  static constexpr int FIELD = NG * GS;
  static constexpr int STAGE = (1 + NO) * FIELD + NG * VS;
};

#ifndef DV3_STAGES
#define DV3_STAGES 2
#endif
#ifndef DV3_U
#define DV3_U 4
#endif
#ifndef DV3_UPHI
#define DV3_UPHI 4
#endif
#ifndef DV3_MINB
#define DV3_MINB 2
#endif
#ifndef DV3_DIV_SPREAD
#define DV3_DIV_SPREAD 1
#endif
#ifndef DV3_MINB_NO1
#define DV3_MINB_NO1 3  // one gathered mode (memo piece sums: 80 registers, 3 CTAs per SM)
#endif
#ifndef DV3_MINB_PHI
#define DV3_MINB_PHI 2
#endif
constexpr int kDv3Stages = DV3_STAGES;

#ifndef DV3_BLOCK
#define DV3_BLOCK 256  // MTTKRP block size (Phi uses 256)
#endif
template <int NO, int G>
constexpr int dv3_smem_bytes(int block) {
  return Dv3Smem<NO, G>::STAGE * kDv3Stages * (block / 32);
}

// Interleaved ("IL") streams (memo_sums.cu): the logical stream (a group of G
// lanes walks one 512-nonzero segment) stored so that one warp's stage --
// quad k of chunk c of each of its NG = 32/G segments -- is one contiguous
// block per field: a warp stages a chunk with one 1D bulk copy (TMA) per
// field instead of per-lane cp.async, and every shared read of a quad serves
// the NG groups from 128 contiguous bytes. Element x of segment seg = x / 512 (warp block
// wb = seg / NG, group g = seg % NG, offset o = x % 512 = c * CH + 4 * k + e,
// CH = 4 G nonzeros per group chunk) lives at
//   u32 fields: wb * NG * 512 + c * 128 + k * 4 NG + g * 4 + e
//   values:     wb * NG * 512 + c * 128 + k * 4 NG + (e / 2) * 2 NG + g * 2 + e % 2
// and the arrays are zero-padded to whole warp blocks (il_len).
constexpr int kIlWarpChunk = 128;  // nonzeros per warp stage (NG groups x CH)
__host__ __device__ inline int64_t il_len(int64_t M, int G) {
  const int64_t blk = (int64_t)(32 / G) * kDvSeg;
  return (M + blk - 1) / blk * blk;
}
template <int G>
__host__ __device__ inline int64_t il_u32(int64_t x) {
  constexpr int NG = 32 / G, CH = 4 * G;
  const int64_t seg = x / kDvSeg;
  const int o = (int)(x % kDvSeg);
  const int c = o / CH, r = o % CH;
  return (seg / NG) * (NG * kDvSeg) + c * kIlWarpChunk + (r >> 2) * 4 * NG + (seg % NG) * 4 + (r & 3);
}
template <int G>
__host__ __device__ inline int64_t il_f64(int64_t x) {
  constexpr int NG = 32 / G, CH = 4 * G;
  const int64_t seg = x / kDvSeg;
  const int o = (int)(x % kDvSeg);
  const int c = o / CH, r = o % CH, e = r & 3;
  return (seg / NG) * (NG * kDvSeg) + c * kIlWarpChunk + (r >> 2) * 4 * NG + (e >> 1) * 2 * NG + (seg % NG) * 2 +
         (e & 1);
}

// LL (with PHI): Poisson log-likelihood data term instead of Phi: `scaled`
// holds lambda o A_mode, d = <scaled[row], krp> = mhat, and the kernel sums
// v * log(mhat) (one lane per group) into per-block partials in a.out.
// End-of-segment flush shared by the dview3 kernels. When every group of
// the warp ends in the same row (a long row spanning all 32/G segments of
// the warp), each group's run of it is an edge run (it continues into the
// next segment or from the previous one): the runs are summed across the
// groups with a fixed shuffle tree and reduced once by group 0 instead of
// 32/G fp64 reductions of the same addresses (which serialise in L2).
template <int G, int VEC, bool DET = false, typename Flush>
__device__ __forceinline__ void dv3_final_flush(uint32_t cur, double (&acc)[VEC], const bool (&colok)[VEC],
                                                bool lane_active, int colv, int lane, const DViewArgs &a,
                                                Flush &&flush) {
  constexpr uint32_t kNone = 0xffffffffu;
#ifndef DV3_NO_WARP_FLUSH
  if constexpr (G < 32) {
    const uint32_t r0 = __shfl_sync(0xffffffffu, cur, 0);
    if (!DET && __all_sync(0xffffffffu, cur == r0 && cur != kNone)) {
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
      return;
    }
  }
#endif
  if (cur != kNone) flush(cur, true);
}

// Predicated 256-bit gather: when !pred no request is issued and the
// registers keep their previous contents.
__device__ __forceinline__ void load_row_if(const double *p, bool pred, double (&r)[4]) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t@q ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];\n\t}"
      : "+d"(r[0]), "+d"(r[1]), "+d"(r[2]), "+d"(r[3])
      : "l"(p), "r"((int)pred));
}

// predicated streaming 256-bit store (no branch, no request when the
// predicate is false)
__device__ __forceinline__ void st_cs_v4_if(double *p, bool pred, const double (&v)[4]) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t@q st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};\n\t}" ::"l"(p),
      "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3]), "r"((int)pred)
      : "memory");
}

}  // namespace alto
