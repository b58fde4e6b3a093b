"""Memoised sweep kernels on c2 (for ncu capture): memo0 (mode 0 + T) and memo1 (mode 1 from T)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic
from paper_2403_06348_b200.cpd import als as ALS
cfg = synthetic.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
c, v = synthetic.generate(cfg, seed=0)
t = alto.AltoTensor.from_device_coo(cfg.dims, c, v)
del c, v
st = ALS.AlsState(t, alto.CpAlsConfig(rank=cfg.rank, max_iters=1, seed=0))
for _ in range(2):
    for n in range(3):
        st.mttkrp(n)
torch.cuda.synchronize()
print("pieces", st._memo().P, "nnz", t.nnz)
