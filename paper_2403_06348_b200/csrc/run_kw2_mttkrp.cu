// Template instantiations: 2-word keys, MTTKRP.
#define RUN_KW 2
#define RUN_PHI 0
#define RUN_ENTRY launch_run_kw2_mttkrp
#include "run_inst.cuh"
