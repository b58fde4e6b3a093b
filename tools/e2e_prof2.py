"""cProfile of the bench's e2e loop (public mttkrp, numpy factors in pinned
memory evolving like a CP-ALS loop, call memo on): host time per call
outside the stream synchronisation."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic
cfg = synthetic.CONFIGS["c2"]
c, v = synthetic.generate(cfg, seed=0)
t = alto.AltoTensor.from_device_coo(cfg.dims, c, v); del c, v
R, N, KV = cfg.rank, 3, 4
rng = np.random.default_rng(1)
hv = []
for d in cfg.dims:
    vers = []
    for _ in range(KV):
        b = torch.empty((d, R), dtype=torch.float64, pin_memory=True)
        b.copy_(torch.from_numpy(rng.random((d, R))))
        vers.append(b.numpy())
    hv.append(vers)
sw = [0]
def sweep():
    s = sw[0]
    for n in range(N):
        alto.mttkrp(t, [hv[m][(s + (1 if m < n else 0)) % KV] for m in range(N)], n)
    sw[0] += 1
for _ in range(4):
    sweep()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    sweep()
print("step ms", (time.perf_counter() - t0) / 20 * 1e3)
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    sweep()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
