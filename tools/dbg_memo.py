import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import kernels as K, _native as nat
from paper_2403_06348_b200.memo import MemoPlan
from oracle import alto_oracle as orc
from conftest import random_sparse
rng = np.random.default_rng(21)
dims = (30, 25, 40)
coords, vals = random_sparse(rng, dims, 3000, kind="positive")
t = alto.AltoTensor.from_coo(alto.CooTensor(dims, coords, vals))
_k, sv, sc = orc.from_coo(dims, *orc.canonicalize(coords, vals))
for R in (1, 2, 3, 4, 5, 8, 16):
    fac = [rng.random((d, R)) for d in dims]
    d = K.DeviceFactors(fac, R)
    for split in ("0", "1"):
        os.environ["ALTO_B200_MEMO_SPLIT"] = split
        errs = []
        for (m0, m1) in ((0, 1), (1, 2), (2, 0)):
            p = MemoPlan(t, R, m0, m1)
            o0 = torch.zeros((dims[m0], nat.padded_ld(R)), dtype=torch.float64, device="cuda")
            o1 = torch.zeros((dims[m1], nat.padded_ld(R)), dtype=torch.float64, device="cuda")
            p.mttkrp_m0(t, d, o0); p.mttkrp_m1(d, o1)
            w0 = orc.mttkrp(sc, sv, fac, m0); w1 = orc.mttkrp(sc, sv, fac, m1)
            errs.append((float(np.abs(o0[:, :R].cpu().numpy() - w0).max() / np.abs(w0).max()),
                         float(np.abs(o1[:, :R].cpu().numpy() - w1).max() / np.abs(w1).max())))
        print(R, split, [f"{a:.1e}/{b:.1e}" for a, b in errs])
