// Fiber-kernel instantiations: included by fiber_kw{1,2}.cu with FIBER_KW set.
#include "fiber_kernels.cuh"

namespace alto {

template <int NM, int G>
static int fiber_one(const RunArgs &a, bool phi, int grid, cudaStream_t st) {
  if (phi)
    fiber_kernel<NM, G, FIBER_KW, true><<<grid, 256, 0, st>>>(a);
  else
    fiber_kernel<NM, G, FIBER_KW, false><<<grid, 256, 0, st>>>(a);
  ALTO_LAUNCH_CHECK("fiber_kernel");
  return ALTO_OK;
}

template <int NM>
static int fiber_g(const RunArgs &a, int g, bool phi, int grid, cudaStream_t st) {
  switch (g) {
    case 1: return fiber_one<NM, 1>(a, phi, grid, st);
    case 2: return fiber_one<NM, 2>(a, phi, grid, st);
    case 4: return fiber_one<NM, 4>(a, phi, grid, st);
    default: return fiber_one<NM, 8>(a, phi, grid, st);
  }
}

int FIBER_ENTRY(const RunArgs &a, int nm, int g, bool phi, int grid, cudaStream_t st) {
  switch (nm) {
    case 3: return fiber_g<3>(a, g, phi, grid, st);
    case 4: return fiber_g<4>(a, g, phi, grid, st);
    case 5: return fiber_g<5>(a, g, phi, grid, st);
    default: set_error("fiber kernels need 3..5 modes"); return ALTO_ERR_UNSUPPORTED;
  }
}

}  // namespace alto
