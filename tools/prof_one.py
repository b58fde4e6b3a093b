"""Run a few MTTKRP/Phi launches on a synthetic config for ncu capture."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic, kernels as K
from paper_2403_06348_b200.cpd import apr as A
cfg = synthetic.CONFIGS[sys.argv[1]]
nnz = int(float(sys.argv[2]))
kern = sys.argv[3]
op = sys.argv[4] if len(sys.argv) > 4 else "mttkrp"
coords, vals = synthetic.generate(cfg, seed=0, nnz=nnz)
t = alto.AltoTensor.from_device_coo(cfg.dims, coords, vals)
del coords
R = cfg.rank
fac = [torch.rand((d, R), dtype=torch.float64, device="cuda") for d in cfg.dims]
dfac = K.DeviceFactors(fac, R)
for mode in range(len(cfg.dims)):
    if op == "mttkrp":
        for _ in range(2):
            K.launch_mttkrp(t, dfac, mode, kern)
    else:
        b = torch.rand((cfg.dims[mode], K.nat.padded_ld(R)), dtype=torch.float64, device="cuda")
        for _ in range(2):
            A.launch_phi(t, dfac, mode, kern, b, 1e-10)
torch.cuda.synchronize()
print("done")
