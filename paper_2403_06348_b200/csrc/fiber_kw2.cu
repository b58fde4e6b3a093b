// Fiber kernel instantiations, 2-word keys.
#define FIBER_KW 2
#define FIBER_ENTRY launch_fiber_kw2
#include "fiber_inst.cuh"
