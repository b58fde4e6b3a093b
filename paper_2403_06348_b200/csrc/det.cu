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
// lanes stride over the chain's segments, a fixed shuffle tree sums them
// (measured 3.57 ms per c2 sweep vs 4.04 with lane = column and the chain
// summed sequentially: the hottest c2 rows span ~10^4 segments).
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
  int64_t e = -1;     // last segment of the chain
  for (int64_t base = s + 1; e < 0; base += 32) {
    const int64_t k = base + lane;
    const bool stop = k >= nseg || through[k] == 0;
    const unsigned m = __ballot_sync(0xffffffffu, stop);
    if (m) e = base + __ffs(m) - 1;
  }
  if (e >= nseg) e = nseg - 1;
  for (int c = 0; c < rank; ++c) {
    double acc = 0.0;
    for (int64_t k = s + 1 + lane; k <= e; k += 32) acc += val[(2 * k) * kDetCols + c];
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[r * ldo + col0 + c] = val[(2 * s + 1) * kDetCols + c] + acc;
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
