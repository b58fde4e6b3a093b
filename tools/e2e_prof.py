"""Break down the public mttkrp() call with host (pinned) numpy factors on c2."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic, kernels as K
from paper_2403_06348_b200 import _native as nat
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
plain = [np.array(h) for h in host]
for n in range(3):
    alto.mttkrp(t, host, n)
torch.cuda.synchronize()
def tm(name, fn, reps=5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): r = fn()
    torch.cuda.synchronize(); print(name, round((time.perf_counter() - t0) / reps * 1e3, 3), "ms", flush=True)
    return r
tm("public mttkrp pinned (mode 0)", lambda: alto.mttkrp(t, host, 0))
tm("public mttkrp pageable (mode 0)", lambda: alto.mttkrp(t, plain, 0))
tm("DeviceFactors(pinned)", lambda: K.DeviceFactors(host, R))
tm("DeviceFactors(pageable)", lambda: K.DeviceFactors(plain, R))
d = K.DeviceFactors(host, R)
o = tm("launch_mttkrp", lambda: K.launch_mttkrp(t, d, 0, "dview"))
tm("result .cpu().numpy()", lambda: o[:, :R].cpu().numpy().copy())
tm("resolve_strategy", lambda: K.resolve_strategy(t, 0, 1, R, 1, "auto", K.DEFAULT_TEMP_BUDGET_BYTES))
print("is_pinned", torch.from_numpy(host[0]).is_pinned())
for n in range(3):
    tm(f"public mttkrp pinned (mode {n})", lambda: alto.mttkrp(t, host, n))
def loop():
    for n in range(3):
        out = alto.mttkrp(t, host, n)
tm("bench-style loop (3 modes)", loop)
import cProfile, pstats
pr = cProfile.Profile(); pr.enable(); loop(); loop(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
