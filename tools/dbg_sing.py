import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2403_06348_b200 as alto
from conftest import random_sparse
rng = np.random.default_rng(21)
dims = (30, 25, 40)
coords, vals = random_sparse(rng, dims, 3000, kind="positive")
t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals))
os.environ["ALTO_B200_KERNEL"] = "dview"
base = alto.init_factors(t.shape, 3, seed=1)
fs = [np.concatenate([f[:, :2], f[:, :1]], axis=1) for f in base.factors]
init = alto.KruskalModel(np.ones(3), fs)
cfg3 = alto.CpAlsConfig(rank=3, max_iters=3, fit_tol=1e-300, seed=1)
for split in ("0", "1"):
    for host in ("0", "1"):
        for memo in ("1", "0"):
            os.environ["ALTO_B200_MEMO_SPLIT"] = split
            os.environ["ALTO_B200_HOST_ALS"] = host
            os.environ["ALTO_B200_MEMO"] = memo
            r = alto.cp_als(alto.AltoTensor(t.layout, t._keys, t._vals, _validate=False), cfg3, init=init)
            print(f"split={split} host={host} memo={memo}", r.fit_trace)
