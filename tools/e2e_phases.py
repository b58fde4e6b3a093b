"""Host-side phase times of the public mttkrp() call (numpy factors in pinned
memory) on c2: where the end-to-end time beyond the kernel goes."""
import os, sys, time, statistics
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
ph = {k: [] for k in ("prepare", "strategy", "factors", "launch", "finish", "total", "gpu_kernel")}
for rep in range(20):
    for mode in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        factors, rank = K._prepare(t, host, mode)
        t1 = time.perf_counter()
        choice = K.resolve_strategy(t, mode, 1, rank, 1, "auto", K.DEFAULT_TEMP_BUDGET_BYTES)
        kernel = K.kernel_for(choice, False)
        t2 = time.perf_counter()
        dfac = K.DeviceFactors(factors, rank, check_finite=True, skip=mode, defer=True, staging=t._cache)
        t3 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        dout = K.launch_mttkrp(t, dfac, mode, kernel, out=t._cache.get(("out", mode, rank)))
        e1.record()
        t4 = time.perf_counter()
        res = K._finish(dout, rank, False, dfac)
        t5 = time.perf_counter()
        if rep >= 5:
            for k, a, b in (("prepare", t0, t1), ("strategy", t1, t2), ("factors", t2, t3), ("launch", t3, t4),
                            ("finish", t4, t5), ("total", t0, t5)):
                ph[k].append((b - a) * 1e3)
            ph["gpu_kernel"].append(e0.elapsed_time(e1))
for k, vals in ph.items():
    print(f"{k:10s} {statistics.mean(vals):.4f} ms")
def loop():
    for n in range(3):
        alto.mttkrp(t, host, n)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(10): loop()
print("step (3 calls)", (time.perf_counter() - t0) / 10 * 1e3, "ms")
