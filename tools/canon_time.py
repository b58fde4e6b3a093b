import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic
# duplicate-heavy COO: 20M draws over a small hot set + unique tail
rng = np.random.default_rng(0)
dims = (2000, 2000, 2000)
M = 20_000_000
z = [np.minimum(rng.zipf(1.5, M) - 1, d - 1) for d in dims]
coords = np.stack(z, axis=1).astype(np.int64); vals = rng.random(M)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    coo = alto.CooTensor(dims, coords, vals)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print("canonicalise 20M draws (zipf 1.5 duplicates): %.1f ms, unique %d" % ((t1 - t0) * 1e3, coo.nnz), flush=True)
cfg = synthetic.CONFIGS["c2"]
torch.cuda.synchronize(); t0 = time.perf_counter()
c, v = synthetic.generate(cfg, seed=0)
torch.cuda.synchronize(); print("generate c2: %.1f ms" % ((time.perf_counter() - t0) * 1e3))
