"""Where a CP-ALS iteration's wall time goes on c2 (device sweep + fit + host)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic
from paper_2403_06348_b200.cpd import als as ALS
cfg = synthetic.CONFIGS["c2"]
c, v = synthetic.generate(cfg, seed=0)
t = alto.AltoTensor.from_device_coo(cfg.dims, c, v); del c, v
st = ALS.AlsState(t, alto.CpAlsConfig(rank=16, max_iters=10, fit_tol=1e-300, seed=0))
for _ in range(4):
    st.sweep(); st.fit()
torch.cuda.synchronize()
def timeit(f, n=20):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3
print("sweep only (no sync) ms", timeit(lambda: st.sweep()))
print("sweep + sync ms", timeit(lambda: (st.sweep(), torch.cuda.synchronize())))
print("sweep + fit ms", timeit(lambda: (st.sweep(), st.fit())))
print("fit only ms", timeit(lambda: st.fit()))
t0 = time.perf_counter(); r = alto.cp_als(t, alto.CpAlsConfig(rank=16, max_iters=10, fit_tol=1e-300, seed=0)); print("cp_als warm s", time.perf_counter() - t0)
