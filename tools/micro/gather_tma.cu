// Micro-benchmark: random 128-byte row gathers with the TMA gather4 mode
// (cp.async.bulk.tensor.2d.tile::gather4, sm_100a) vs the LSU path
// (256-bit loads, 8 rows per warp-wide load) -- does the TMA unit gather
// factor rows faster than the L1TEX path that bounds the decoded-view kernels?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_tma gather_tma.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

constexpr int kWarps = 8;
constexpr int kDepth = 16;  // gather4 requests in flight per warp
constexpr int kSlotBytes = 4 * 128;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(kWarps * 32, 1)
    tma_gather_kernel(const __grid_constant__ CUtensorMap tm, const uint32_t *__restrict__ idx, int64_t nquads,
                      uint32_t rows, double *out) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bars[kWarps][kDepth];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char *ring = smem + (size_t)w * kDepth * kSlotBytes;
  if (lane == 0) {
    for (int s = 0; s < kDepth; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[w][s])) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncwarp();
  const int64_t gw = (int64_t)blockIdx.x * kWarps + w, nw = (int64_t)gridDim.x * kWarps;
  const int64_t my = gw < nquads ? (nquads - gw + nw - 1) / nw : 0;
  auto issue = [&](int64_t i) {
    const int s = (int)(i % kDepth);
    const int64_t q = gw + i * nw;
    const uint32_t *p = idx + 4 * q;
    const int32_t r0 = (int32_t)(p[0] % rows), r1 = (int32_t)(p[1] % rows), r2 = (int32_t)(p[2] % rows),
                  r3 = (int32_t)(p[3] % rows);
    const uint32_t bar = smem_u32(&bars[w][s]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kSlotBytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
        "%4, %5, %6}], [%7];" ::"r"(smem_u32(ring + (size_t)s * kSlotBytes)),
        "l"(&tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
        : "memory");
  };
  double acc = 0.0;
  if (lane == 0)
    for (int64_t i = 0; i < kDepth && i < my; ++i) issue(i);
  for (int64_t i = 0; i < my; ++i) {
    const int s = (int)(i % kDepth);
    const uint32_t parity = (uint32_t)((i / kDepth) & 1);
    asm volatile(
        "{\n\t.reg .pred P;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}" ::"r"(
            smem_u32(&bars[w][s])),
        "r"(parity)
        : "memory");
    acc += reinterpret_cast<const double *>(ring + (size_t)s * kSlotBytes)[lane * 2];
    __syncwarp();
    if (lane == 0 && i + kDepth < my) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(i + kDepth);
    }
  }
  if (acc == 1.2345e-300) out[0] = acc;
}

__global__ void __launch_bounds__(256, 2) lsu_gather_kernel(const double *__restrict__ tab,
                                                           const uint32_t *__restrict__ idx, int64_t n,
                                                           uint32_t rows, double *out) {
  const int lane = threadIdx.x & 31, grp = lane >> 2, gl = lane & 3;
  double acc[4] = {0, 0, 0, 0};
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp * 32; base + 32 <= n; base += nwarps * 32) {
    double f[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t r = idx[base + u * 8 + grp] % rows;
      const double *p = tab + (uint64_t)r * 16 + gl * 4;
      asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                   : "=d"(f[u][0]), "=d"(f[u][1]), "=d"(f[u][2]), "=d"(f[u][3])
                   : "l"(p));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[v] += f[u][v];
  }
  if (acc[0] + acc[1] + acc[2] + acc[3] == 1.2345e-300) out[0] = acc[0];
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t nidx = (int64_t)1 << 26;
  uint32_t *idx;
  double *out;
  cudaMalloc(&idx, nidx * 4);
  cudaMalloc(&out, 64);
  uint32_t *h = (uint32_t *)malloc(nidx * 4);
  uint64_t s = 88172645463325252ull;
  for (int64_t i = 0; i < nidx; ++i) {
    s ^= s << 13;
    s ^= s >> 7;
    s ^= s << 17;
    h[i] = (uint32_t)s;
  }
  cudaMemcpy(idx, h, nidx * 4, cudaMemcpyHostToDevice);
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&encode, cudaEnableDefault, &qr);
  if (!encode) {
    printf("no cuTensorMapEncodeTiled\n");
    return 1;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const uint32_t rows_list[] = {512, 28000, 200000, 2000000};
  for (uint32_t rows : rows_list) {
    double *tab;
    cudaMalloc(&tab, (size_t)rows * 128);
    cudaMemset(tab, 0, (size_t)rows * 128);
    CUtensorMap tm;
    cuuint64_t gdim[2] = {16, rows};
    cuuint64_t gstride[1] = {128};
    cuuint32_t box[2] = {16, 1};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, tab, gdim, gstride, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("encode failed %d\n", (int)r);
      return 1;
    }
    const int64_t nquads = nidx / 4;
    const size_t smem = (size_t)kWarps * kDepth * kSlotBytes;
    cudaFuncSetAttribute(tma_gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int grid_mult = 1; grid_mult <= 3; ++grid_mult) {
      const int grid = sms * grid_mult;
      tma_gather_kernel<<<grid, kWarps * 32, smem>>>(tm, idx, nquads, rows, out);
      cudaEventRecord(e0);
      for (int it = 0; it < 5; ++it) tma_gather_kernel<<<grid, kWarps * 32, smem>>>(tm, idx, nquads, rows, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 5;
      printf("{\"path\": \"tma_gather4\", \"rows\": %u, \"ctas_per_sm\": %d, \"ms\": %.4f, \"GBps\": %.1f, \"err\": \"%s\"}\n",
             rows, grid_mult, ms, (double)nquads * 512 / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
    }
    lsu_gather_kernel<<<sms * 2, 256>>>(tab, idx, nidx, rows, out);
    cudaEventRecord(e0);
    for (int it = 0; it < 5; ++it) lsu_gather_kernel<<<sms * 2, 256>>>(tab, idx, nidx, rows, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    // lsu: a warp visits 4 x 8 rows per 32 indices -> nidx rows
    printf("{\"path\": \"lsu_ldg256\", \"rows\": %u, \"ms\": %.4f, \"GBps\": %.1f}\n", rows, ms,
           (double)nidx * 128 / (ms * 1e6));
    cudaFree(tab);
  }
  return 0;
}
