// Micro-benchmark: L1TEX cost of 128-byte row gathers from a table that is
// L1/L2 resident, by how many distinct rows one warp-wide LDG touches.
//   mode 0: 4 lanes x 32 B per row, 8 rows per LDG.256 (dview3's pattern)
//   mode 1: the same loads split into 8 predicated LDGs, one row each
//   mode 2: 8 lanes x 16 B per row, 4 rows per LDG.128
//   mode 3: 2 lanes x 64 B per row (two LDG.256 per lane, adjacent sectors), 16 rows per LDG pair
//   mode 4: 2 lanes x 64 B per row, lane sectors interleaved (lane 0: sectors 0 and 2, lane 1: 1 and 3)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_wf gather_wf.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld256(const double *p, double (&r)[4]) {
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3]) : "l"(p));
}

template <int MODE>
__global__ void __launch_bounds__(256, 2) gk(const double *__restrict__ tab, const uint32_t *__restrict__ idx,
                                           int64_t n, uint32_t rows, double *out) {
  const int lane = threadIdx.x & 31;
  double acc[4] = {0, 0, 0, 0};
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  constexpr int U = 4;
  for (int64_t base = warp * 32 * U; base < n; base += nwarps * 32 * U) {
    double f[U][4];
    if (MODE == 0 || MODE == 1) {
      const int grp = lane >> 2, gl = lane & 3;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t r = idx[base + u * 8 + grp] % rows;
        const double *p = tab + (uint64_t)r * 16 + gl * 4;
        if (MODE == 0) {
          ld256(p, f[u]);
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (grp == q) ld256(p, f[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[v] += f[u][v];
    } else if (MODE == 3 || MODE == 4) {
      const int grp = lane >> 1, gl = lane & 1;
      double g2[U][4];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t r = idx[base + u * 16 + grp] % rows;
        const double *p = tab + (uint64_t)r * 16 + (MODE == 3 ? gl * 8 : gl * 4);
        ld256(p, f[u]);
        ld256(p + (MODE == 3 ? 4 : 8), g2[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[v] += f[u][v] + g2[u][v];
    } else {
      const int grp = lane >> 3, gl = lane & 7;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t r = idx[base + u * 4 + grp] % rows;
        const double2 t = __ldg(reinterpret_cast<const double2 *>(tab + (uint64_t)r * 16 + gl * 2));
        f[u][0] = t.x; f[u][1] = t.y; f[u][2] = 0; f[u][3] = 0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[v] += f[u][v];
    }
  }
  if (acc[0] + acc[1] + acc[2] + acc[3] == 12345.678) out[0] = acc[0];
}

int main() {
  const int64_t n = 1 << 26;  // row visits
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *tab, *out;
  uint32_t *idx;
  cudaMalloc(&tab, (size_t)1 << 26);
  cudaMalloc(&out, 64);
  cudaMalloc(&idx, n * 4 + 4096);
  cudaMemset(tab, 0, (size_t)1 << 26);
  uint32_t *h = (uint32_t *)malloc(n * 4 + 4096);
  uint64_t s = 88172645463325252ull;
  for (int64_t i = 0; i < n + 1024; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (uint32_t)s; }
  cudaMemcpy(idx, h, n * 4 + 4096, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const uint32_t rows_list[] = {512, 1024, 9000, 28000, 200000};
  for (uint32_t rows : rows_list) {
    for (int mode = 0; mode < 5; ++mode) {
      auto launch = [&]() {
        if (mode == 0) gk<0><<<sms * 2, 256>>>(tab, idx, n, rows, out);
        else if (mode == 1) gk<1><<<sms * 2, 256>>>(tab, idx, n, rows, out);
        else if (mode == 2) gk<2><<<sms * 2, 256>>>(tab, idx, n, rows, out);
        else if (mode == 3) gk<3><<<sms * 2, 256>>>(tab, idx, n, rows, out);
        else gk<4><<<sms * 2, 256>>>(tab, idx, n, rows, out);
      };
      launch();
      cudaEventRecord(e0);
      for (int it = 0; it < 5; ++it) launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 5;
      // row visits: mode 0/1: n (8 rows per 32 idx), mode 2: n (4 rows per... same count of idx reads)
      const double visits = mode == 2 ? (double)n / 8 : (mode >= 3 ? (double)n / 2 : (double)n / 4);  // rows gathered per launch
      printf("{\"rows\": %u, \"mode\": %d, \"ms\": %.4f, \"Grows_per_s\": %.2f, \"cyc_per_row_per_sm\": %.3f}\n",
             rows, mode, ms, visits / ms / 1e6, (ms * 1e-3 * 1.965e9 * sms) / visits);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
