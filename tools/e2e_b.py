import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic
from paper_2403_06348_b200.cpd import als as ALS
cfg = synthetic.CONFIGS["c2"]
c, v = synthetic.generate(cfg, seed=0)
t = alto.AltoTensor.from_device_coo(cfg.dims, c, v); del c, v
R = cfg.rank
rng = np.random.default_rng(1)
host = []
for d in cfg.dims:
    buf = torch.empty((d, R), dtype=torch.float64, pin_memory=True)
    buf.copy_(torch.from_numpy(rng.random((d, R))))
    host.append(buf.numpy())
def loop():
    for n in range(3):
        out = alto.mttkrp(t, host, n)
def tm(name, fn, reps=5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); print(name, round((time.perf_counter() - t0) / reps * 1e3, 3), "ms", flush=True)
loop(); tm("loop before ALS", loop)
st = ALS.AlsState(t, alto.CpAlsConfig(rank=R, max_iters=10, fit_tol=1e-300, seed=0))
for _ in range(5): st.sweep()
torch.cuda.synchronize()
tm("loop after ALS", loop)
del st; torch.cuda.empty_cache()
tm("loop after ALS freed", loop)
