// Instantiation helper: included by run_kw{1,2}_{mttkrp,phi}.cu with
// RUN_KW (1|2) and RUN_PHI (0|1) defined.
#include "run_kernels.cuh"

namespace alto {

template <int NM, int G>
static int launch_one(const RunArgs &a, bool exact, bool atomic, int grid, cudaStream_t st) {
  constexpr bool PHI = RUN_PHI != 0;
  if (atomic)
    run_kernel<NM, G, kVec, RUN_KW, PHI, false, true><<<grid, 256, 0, st>>>(a);
  else if (exact)
    run_kernel<NM, G, kVec, RUN_KW, PHI, true, false><<<grid, 256, 0, st>>>(a);
  else
    run_kernel<NM, G, kVec, RUN_KW, PHI, false, false><<<grid, 256, 0, st>>>(a);
  ALTO_LAUNCH_CHECK("run_kernel");
  return ALTO_OK;
}

template <int NM>
static int launch_g(const RunArgs &a, int g, bool exact, bool atomic, int grid, cudaStream_t st) {
  switch (g) {
    case 1: return launch_one<NM, 1>(a, exact, atomic, grid, st);
    case 2: return launch_one<NM, 2>(a, exact, atomic, grid, st);
    case 4: return launch_one<NM, 4>(a, exact, atomic, grid, st);
    case 8: return launch_one<NM, 8>(a, exact, atomic, grid, st);
    default:
      if constexpr (kVec * 16 <= kMaxRankChunk) return launch_one<NM, 16>(a, exact, atomic, grid, st);
      else return launch_one<NM, 8>(a, exact, atomic, grid, st);
  }
}

int RUN_ENTRY(const RunArgs &a, int nm, int g, bool exact, bool atomic, int grid, cudaStream_t st) {
  switch (nm) {
    case 3: return launch_g<3>(a, g, exact, atomic, grid, st);
    case 4: return launch_g<4>(a, g, exact, atomic, grid, st);
    case 5: return launch_g<5>(a, g, exact, atomic, grid, st);
    default: return launch_g<0>(a, g, exact, atomic, grid, st);
  }
}

}  // namespace alto
