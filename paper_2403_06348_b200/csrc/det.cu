// Deterministic mode of the fast row-run kernels (dview3, memo0, memo1).
//
// The fast kernels accumulate every row run in registers and write it with a
// plain store, except the runs cut by a 512-nonzero segment edge: those are
// reduced with red.global.add.f64, whose order varies from run to run. With
// the deterministic mode on, an edge run is parked instead in a per-segment
// slot (slot 0: the segment's first run, continued from the left; slot 1:
// its last run, continued to the right; a segment that is one run of a row
// crossing it on both sides is flagged "through"), and det_merge_kernel then
// folds every chain -- the head segment's slot 1 plus slot 0 of the
// following segments up to the first that is not "through" -- in a fixed
// order and stores the row once. Same scheme as the exact output-oriented
// merge (run.cu, merge_edges_kernel), made warp-parallel over the chain:
// every lane sums a contiguous block of the chain's slots with vector loads,
// a fixed shuffle tree combines the lanes (the hottest c2 rows span ~10^4
// segments).
// Results are bitwise reproducible run to run (not bitwise equal to the
// reference's order: that is exact=True).
#include "det.cuh"

namespace alto {

static bool g_det = false;
static DetEdges g_edges{nullptr, nullptr, nullptr};
static int64_t g_cap = 0;

bool det_enabled() { return g_det; }

__global__ void det_merge_kernel(int64_t nseg, const int64_t *__restrict__ row, const int32_t *__restrict__ through,
                                 const double *__restrict__ val, double *__restrict__ out, int64_t ldo, int32_t col0,
                                 int32_t rank) {
  const int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= nseg) return;
  const int64_t r = row[2 * s + 1];
  if (r < 0) return;  // warp-uniform: no chain starts here
  int64_t e = -1;     // last segment of the chain: the first one not "through"
  for (int64_t base = s + 1; e < 0; base += 256) {
    // each lane scans 8 consecutive flags: 256 segments per step
    int first = 8;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t k = base + lane * 8 + i;
      if (first == 8 && (k >= nseg || through[k] == 0)) first = i;
    }
    const unsigned m = __ballot_sync(0xffffffffu, first < 8);
    if (m) {
      const int src = __ffs(m) - 1;
      e = base + src * 8 + __shfl_sync(0xffffffffu, first, src);
    }
  }
  if (e >= nseg) e = nseg - 1;
  // lane l sums a contiguous block of the chain's slots in ascending order
  // (8 columns per pass, two 256-bit loads per slot), then a fixed xor tree
  // over the lanes: deterministic, and a chain of 10^4 segments costs each
  // lane ~300 independent vector loads
  const int64_t n = e - s, per = (n + 31) / 32;
  const int64_t k0 = s + 1 + lane * per, k1 = k0 + per <= e + 1 ? k0 + per : e + 1;
  for (int c0 = 0; c0 < rank; c0 += 8) {
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int64_t k = k0;
    for (; k + 4 <= k1; k += 4) {  // four slots' loads in flight, added in order
      double4 x[4], y[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double4 *p = reinterpret_cast<const double4 *>(val + (2 * (k + i)) * kDetCols + c0);
        x[i] = p[0];
        y[i] = p[1];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[0] += x[i].x, acc[1] += x[i].y, acc[2] += x[i].z, acc[3] += x[i].w;
        acc[4] += y[i].x, acc[5] += y[i].y, acc[6] += y[i].z, acc[7] += y[i].w;
      }
    }
    for (; k < k1; ++k) {
      const double4 *p = reinterpret_cast<const double4 *>(val + (2 * k) * kDetCols + c0);
      const double4 x = p[0], y = p[1];
      acc[0] += x.x, acc[1] += x.y, acc[2] += x.z, acc[3] += x.w;
      acc[4] += y.x, acc[5] += y.y, acc[6] += y.z, acc[7] += y.w;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int o = 16; o; o >>= 1) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
    if (lane < 8 && c0 + lane < rank) {
      double t = acc[0];
#pragma unroll
      for (int i = 1; i < 8; ++i) t = lane == i ? acc[i] : t;
      out[r * ldo + col0 + c0 + lane] = val[(2 * s + 1) * kDetCols + c0 + lane] + t;
    }
  }
}

int det_edges(int64_t nseg, DetEdges *e, cudaStream_t st) {
  if (nseg > g_cap) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    ALTO_CUDA(cudaStreamIsCapturing(st, &cs));
    ALTO_REQUIRE(cs == cudaStreamCaptureStatusNone, ALTO_ERR_UNSUPPORTED,
                 "deterministic edge slots must be sized before graph capture (run one launch eagerly)");
    // the old slots are not freed: captured CUDA graphs may still point at them
    const int64_t cap = nseg + nseg / 4 + 1024;
    ALTO_CUDA(cudaMalloc(&g_edges.row, (size_t)cap * 2 * sizeof(int64_t)));
    ALTO_CUDA(cudaMalloc(&g_edges.through, (size_t)cap * sizeof(int32_t)));
    ALTO_CUDA(cudaMalloc(&g_edges.val, (size_t)cap * 2 * kDetCols * sizeof(double)));
    g_cap = cap;
  }
  ALTO_CUDA(cudaMemsetAsync(g_edges.row, 0xff, (size_t)nseg * 2 * sizeof(int64_t), st));  // -1: no run
  ALTO_CUDA(cudaMemsetAsync(g_edges.through, 0, (size_t)nseg * sizeof(int32_t), st));
  *e = g_edges;
  return ALTO_OK;
}

int det_merge(const DetEdges &e, int64_t nseg, double *out, int64_t ldo, int col0, int rank, cudaStream_t st) {
  const int64_t blocks = (nseg * 32 + 255) / 256;
  det_merge_kernel<<<(int)blocks, 256, 0, st>>>(nseg, e.row, e.through, e.val, out, ldo, col0, rank);
  ALTO_LAUNCH_CHECK("det_merge_kernel");
  return ALTO_OK;
}

}  // namespace alto

extern "C" {

int alto_set_deterministic(int32_t on) {
  alto::g_det = on != 0;
  return ALTO_OK;
}

int alto_get_deterministic(int32_t *host_on) {
  ALTO_REQUIRE(host_on != nullptr, ALTO_ERR_VALUE, "null output");
  *host_on = alto::g_det ? 1 : 0;
  return ALTO_OK;
}

}  // extern "C"
