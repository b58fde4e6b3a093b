// Gather-rate probe: the measured ceiling of the factor-row gathers that
// bound every decoded-view kernel (profiles/r02_memo_split.md). Random
// 128-byte rows of a table, 4 lanes x 32 B per row and 8 rows per warp-wide
// 256-bit load (dview3's pattern), 4 loads in flight per lane, all SMs.
// bench.py runs it on the box it measures and reports the kernels' gathered
// bytes against it next to the HBM roofline.
#include "alto_common.cuh"

namespace alto {
namespace {

__global__ void __launch_bounds__(256, 2) gather_probe_kernel(const double *__restrict__ tab,
                                                              const uint32_t *__restrict__ idx, int64_t n,
                                                              uint32_t rows, double *out) {
  const int lane = threadIdx.x & 31, grp = lane >> 2, gl = lane & 3;
  double acc[4] = {0, 0, 0, 0};
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  constexpr int U = 4;
  for (int64_t base = warp * 32 * U; base + 32 * U <= n; base += nwarps * 32 * U) {
    double f[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t r = idx[base + u * 8 + grp] % rows;
      const double *p = tab + (uint64_t)r * 16 + gl * 4;
      asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                   : "=d"(f[u][0]), "=d"(f[u][1]), "=d"(f[u][2]), "=d"(f[u][3])
                   : "l"(p));
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[v] += f[u][v];
  }
  if (acc[0] + acc[1] + acc[2] + acc[3] == 1.2345e-300) out[0] = acc[0];
}

__global__ void probe_fill_kernel(uint32_t *idx, int64_t n, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t s = seed ^ (0x9E3779B97F4A7C15ull * (uint64_t)(i + 1));
    s ^= s >> 33;
    s *= 0xff51afd7ed558ccdull;
    s ^= s >> 33;
    idx[i] = (uint32_t)s;
  }
}

}  // namespace
}  // namespace alto

using namespace alto;

extern "C" {

int alto_gather_probe(int32_t table_rows, int32_t reps, double *host_rows_per_s) {
  ALTO_REQUIRE(table_rows >= 1 && reps >= 1 && host_rows_per_s != nullptr, ALTO_ERR_VALUE, "bad probe arguments");
  const int64_t n = (int64_t)1 << 26;  // row visits x 4 indices read per 32 lanes
  double *tab = nullptr, *out = nullptr;
  uint32_t *idx = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int rc = ALTO_OK;
  float ms = 0.f;
  const int sms = num_sms();
  do {
    if (cudaMalloc(&tab, (size_t)table_rows * 128) != cudaSuccess || cudaMalloc(&out, 64) != cudaSuccess ||
        cudaMalloc(&idx, (size_t)n * 4) != cudaSuccess) {
      rc = cuda_status(cudaGetLastError(), "probe allocation");
      break;
    }
    cudaMemset(tab, 0, (size_t)table_rows * 128);
    probe_fill_kernel<<<sms * 8, 256>>>(idx, n, 12345);
    gather_probe_kernel<<<sms * 2, 256>>>(tab, idx, n, (uint32_t)table_rows, out);  // warm-up
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) gather_probe_kernel<<<sms * 2, 256>>>(tab, idx, n, (uint32_t)table_rows, out);
    cudaEventRecord(e1);
    if (cudaEventSynchronize(e1) != cudaSuccess) {
      rc = cuda_status(cudaGetLastError(), "gather probe");
      break;
    }
    cudaEventElapsedTime(&ms, e0, e1);
  } while (0);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  cudaFree(tab);
  cudaFree(out);
  cudaFree(idx);
  if (rc) return rc;
  // each warp iteration visits 8 rows per 32 indices: n / 4 rows per launch
  *host_rows_per_s = (double)(n / 4) * reps / (ms * 1e-3);
  return ALTO_OK;
}

}  // extern "C"
