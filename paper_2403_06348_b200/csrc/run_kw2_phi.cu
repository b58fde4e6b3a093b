// Template instantiations: 2-word keys, Phi.
#define RUN_KW 2
#define RUN_PHI 1
#define RUN_ENTRY launch_run_kw2_phi
#include "run_inst.cuh"
