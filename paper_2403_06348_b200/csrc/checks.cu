// Finiteness scan of factor matrices on the device: the factor checks of
// pkg/src/alto/validation.py:30-57 (check_factors: "factor n contains
// non-finite entries") for factors uploaded from host memory, as one
// stream-ordered launch whose flags the caller reads back together with the
// result of the kernel that consumes the factors (no extra host round trip).
#include <math.h>

#include "alto_common.cuh"

namespace alto {
namespace {

struct FiniteArgs {
  const double *ptr[ALTO_MAX_MODES];
  int64_t ld[ALTO_MAX_MODES];
  int64_t rows[ALTO_MAX_MODES];
  int64_t start[ALTO_MAX_MODES + 1];  // prefix of rows * rank over the scanned modes
  int32_t mode[ALTO_MAX_MODES];
  int32_t count;
  int32_t rank;
};

// grid-stride over the concatenated (mode, row, column) index space; a warp
// that sees a non-finite entry sets its mode's flag (plain stores of 1)
__global__ void __launch_bounds__(256) nonfinite_kernel(const __grid_constant__ FiniteArgs a, int32_t *flags) {
  const int64_t total = a.start[a.count];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int k = 0;
    while (k + 1 < a.count && i >= a.start[k + 1]) ++k;
    const int64_t off = i - a.start[k];
    const int64_t r = off / a.rank, c = off - r * a.rank;
    if (!isfinite(a.ptr[k][r * a.ld[k] + c])) flags[a.mode[k]] = 1;
  }
}

}  // namespace
}  // namespace alto

using namespace alto;

extern "C" {

int alto_factors_nonfinite(const alto_factors_t *host_factors, const int64_t *host_rows, int32_t skip,
                           int32_t *flags, void *stream) {
  ALTO_REQUIRE(host_factors && host_rows && flags, ALTO_ERR_VALUE, "null argument");
  const alto_factors_t &F = *host_factors;
  ALTO_REQUIRE(F.nmodes >= 1 && F.nmodes <= ALTO_MAX_MODES, ALTO_ERR_VALUE, "bad mode count %d", F.nmodes);
  ALTO_REQUIRE(F.rank >= 1, ALTO_ERR_VALUE, "rank must be positive");
  cudaStream_t st = (cudaStream_t)stream;
  ALTO_CUDA(cudaMemsetAsync(flags, 0, sizeof(int32_t) * F.nmodes, st));
  FiniteArgs a{};
  a.rank = F.rank;
  int64_t total = 0;
  for (int n = 0; n < F.nmodes; ++n) {
    if (n == skip || host_rows[n] <= 0) continue;
    ALTO_REQUIRE(F.ptr[n] != nullptr && F.ld[n] >= F.rank, ALTO_ERR_VALUE, "bad factor %d", n);
    a.ptr[a.count] = F.ptr[n];
    a.ld[a.count] = F.ld[n];
    a.rows[a.count] = host_rows[n];
    a.mode[a.count] = n;
    a.start[a.count] = total;
    total += host_rows[n] * F.rank;
    ++a.count;
  }
  a.start[a.count] = total;
  if (total == 0) return ALTO_OK;
  const int64_t blocks = ceil_div(total, (int64_t)256);
  const int grid = (int)(blocks < 4 * 148 ? blocks : 4 * 148);
  nonfinite_kernel<<<grid, 256, 0, st>>>(a, flags);
  ALTO_LAUNCH_CHECK("nonfinite_kernel");
  return ALTO_OK;
}

// Host (row-major, `host_ld` doubles per row) -> device factor copies for
// every mode but `skip`, then the finiteness scan above: the whole upload of
// a public numpy-input call in one stream-ordered C call.
int alto_upload_factors(const alto_factors_t *dev_factors, const double *const *host_ptrs, const int64_t *host_rows,
                        int32_t host_ld, int32_t skip, int32_t *flags, void *stream) {
  ALTO_REQUIRE(dev_factors && host_ptrs && host_rows, ALTO_ERR_VALUE, "null argument");
  const alto_factors_t &F = *dev_factors;
  ALTO_REQUIRE(F.nmodes >= 1 && F.nmodes <= ALTO_MAX_MODES, ALTO_ERR_VALUE, "bad mode count %d", F.nmodes);
  ALTO_REQUIRE(host_ld >= F.rank, ALTO_ERR_VALUE, "host row stride %d below the rank %d", host_ld, F.rank);
  cudaStream_t st = (cudaStream_t)stream;
  for (int n = 0; n < F.nmodes; ++n) {
    if (n == skip || host_rows[n] <= 0) continue;
    ALTO_REQUIRE(F.ptr[n] != nullptr && host_ptrs[n] != nullptr && F.ld[n] >= F.rank, ALTO_ERR_VALUE,
                 "bad factor %d", n);
    double *dst = const_cast<double *>(F.ptr[n]);
    if (F.ld[n] == host_ld && host_ld == F.rank) {  // both contiguous: one linear DMA
      ALTO_CUDA(cudaMemcpyAsync(dst, host_ptrs[n], (size_t)host_rows[n] * host_ld * sizeof(double),
                                cudaMemcpyHostToDevice, st));
    } else {
      ALTO_CUDA(cudaMemcpy2DAsync(dst, (size_t)F.ld[n] * sizeof(double), host_ptrs[n],
                                  (size_t)host_ld * sizeof(double), (size_t)F.rank * sizeof(double),
                                  (size_t)host_rows[n], cudaMemcpyHostToDevice, st));
    }
  }
  return flags ? alto_factors_nonfinite(dev_factors, host_rows, skip, flags, stream) : ALTO_OK;
}

int alto_memset_async(void *ptr, size_t bytes, void *stream) {
  if (bytes == 0) return ALTO_OK;
  ALTO_REQUIRE(ptr != nullptr, ALTO_ERR_VALUE, "null pointer");
  ALTO_CUDA(cudaMemsetAsync(ptr, 0, bytes, (cudaStream_t)stream));
  return ALTO_OK;
}

}  // extern "C"
