// Fiber kernel instantiations, 1-word keys.
#define FIBER_KW 1
#define FIBER_ENTRY launch_fiber_kw1
#include "fiber_inst.cuh"
