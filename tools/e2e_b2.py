"""Per-phase timing of the public mttkrp() call per mode (c2, pinned host factors)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic, kernels as K
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
for n in range(3):
    alto.mttkrp(t, host, n)
torch.cuda.synchronize()
for rep in range(3):
    for n in range(3):
        ph = []
        t0 = time.perf_counter()
        f, rank = K._prepare(t, host, n); ph.append(time.perf_counter())
        choice = K.resolve_strategy(t, n, 1, rank, 1, "auto", K.DEFAULT_TEMP_BUDGET_BYTES); ph.append(time.perf_counter())
        kern = K.kernel_for(choice, K.resolve_exact(None)); ph.append(time.perf_counter())
        d = K.DeviceFactors(f, rank, check_finite=True, skip=n); ph.append(time.perf_counter())
        o = K.launch_mttkrp(t, d, n, kern); ph.append(time.perf_counter())
        torch.cuda.synchronize(); ph.append(time.perf_counter())
        r = K._finish(o, rank, False); ph.append(time.perf_counter())
        names = ["prepare", "strategy", "kernel_for", "devfac", "launch", "sync", "finish"]
        prev = t0
        s = []
        for nm, x in zip(names, ph):
            s.append(f"{nm}={1e3*(x-prev):.3f}")
            prev = x
        print(f"mode {n}: total {1e3*(ph[-1]-t0):.3f} ms  " + " ".join(s), flush=True)
