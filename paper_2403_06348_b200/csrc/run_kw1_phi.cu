// Template instantiations: 1-word keys, Phi.
#define RUN_KW 1
#define RUN_PHI 1
#define RUN_ENTRY launch_run_kw1_phi
#include "run_inst.cuh"
