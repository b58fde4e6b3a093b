"""Break down one CP-APR outer iteration on c4 (host timers around synced phases)."""
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
acc = {}
def timed(name, fn):
    def w(*a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize(); acc[name] = acc.get(name, 0) + time.perf_counter() - t0
        return r
    return w
A.launch_phi = timed("phi", A.launch_phi)
A.apr_update = timed("apr_update", A.apr_update)
A.loglik_data_term = timed("loglik", A.loglik_data_term)
torch.cuda.synchronize(); t0 = time.perf_counter()
st.outer(); torch.cuda.synchronize()
tot = time.perf_counter() - t0
print({k: round(v * 1e3, 2) for k, v in acc.items()}, "total ms", round(tot * 1e3, 2), "kernels", st.kernels, flush=True)
