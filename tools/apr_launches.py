"""One CP-APR outer iteration on c4 inside an NVTX range 'apr' (for an ncu launch list),
plus its wall time with events (no profiler)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic
from paper_2403_06348_b200.cpd import apr as A
cfg = synthetic.CONFIGS["c4"]
c, v = synthetic.generate(cfg, seed=0)
t = alto.AltoTensor.from_device_coo(cfg.dims, c, v); del c, v
st = A.AprState(t, alto.CpAprConfig(rank=10, max_outer=5, max_inner=10, eps=1e-10, seed=0))
st.outer(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.nvtx.range_push("apr")
e0.record(); t0 = time.perf_counter()
st.outer()
e1.record(); torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("outer ms (events)", e0.elapsed_time(e1), "wall", (time.perf_counter() - t0) * 1e3, st.inner_counts[-1])
