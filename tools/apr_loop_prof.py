"""Device-driven inner loop vs bare Phi launches on c4 (events, no profiler)."""
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
def ev(fn, reps=3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); h0 = time.perf_counter(); e0.record()
    for _ in range(reps): fn()
    e1.record(); h1 = time.perf_counter(); torch.cuda.synchronize(); h2 = time.perf_counter()
    return round(e0.elapsed_time(e1) / reps, 3), round((h1 - h0) / reps * 1e3, 3), round((h2 - h0) / reps * 1e3, 3)
for n in range(3):
    b = st.b[n]
    out = torch.zeros_like(b)
    print("mode", n, "10x phi (gpu ms, host enqueue ms, wall ms)", ev(lambda: [A.launch_phi(t, st.dfac, n, "dview", b, 1e-10, out=out) for _ in range(10)]))
    state = st._inner_state
    print("mode", n, "update_mode", ev(lambda: st.update_mode(n, 3), reps=1))
print("loglik", ev(lambda: st.loglik()))
print("outer", ev(lambda: st.outer(), reps=1))
