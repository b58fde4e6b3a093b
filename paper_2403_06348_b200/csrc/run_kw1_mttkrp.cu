// Template instantiations: 1-word keys, MTTKRP.
#define RUN_KW 1
#define RUN_PHI 0
#define RUN_ENTRY launch_run_kw1_mttkrp
#include "run_inst.cuh"
