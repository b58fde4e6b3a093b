// Deterministic mode: parked segment-edge runs and their ordered merge
// (det.cu). The kernels park an edge run with det_park instead of an fp64
// reduction when the edge buffers are set.
#pragma once

#include "alto_common.cuh"

namespace alto {

constexpr int kDetCols = 32;  // slot width (columns of one rank chunk)

struct DetEdges {
  int64_t *row;       // [2 * nseg]: slot 0 = first run's row, slot 1 = last run's row, -1 = none
  int32_t *through;   // [nseg]: the segment is one run of a row crossing both its edges
  double *val;        // [2 * nseg][kDetCols]
};

bool det_enabled();
// grow-only edge slots for nseg segments, reset on the stream
int det_edges(int64_t nseg, DetEdges *e, cudaStream_t st);
// fold every chain in a fixed order and store its row (columns col0 .. col0 + rank)
int det_merge(const DetEdges &e, int64_t nseg, double *out, int64_t ldo, int col0, int rank, cudaStream_t st);

// park an edge run of segment `seg` (lane's VEC columns starting at colv)
template <int VEC>
__device__ __forceinline__ void det_park(const DetEdges &e, int64_t seg, bool from_left, bool to_right, uint32_t row,
                                         const double (&acc)[VEC], int colv, int gl, bool lane_active) {
  const int slot = from_left ? 0 : 1;
  if (lane_active) {
    double *p = e.val + (2 * seg + slot) * kDetCols + colv;
#pragma unroll
    for (int v = 0; v < VEC; ++v) p[v] = acc[v];
  }
  if (gl == 0) {
    e.row[2 * seg + slot] = (int64_t)row;
    if (from_left && to_right) e.through[seg] = 1;
  }
}

}  // namespace alto
