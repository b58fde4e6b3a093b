"""Launch the fused memo producer (c2 pair 0 -> 1) and the consumer a few
times (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic, kernels as K, _native as nat
from paper_2403_06348_b200.memo import MemoPlan
cfg = synthetic.CONFIGS["c2"]
c, v = synthetic.generate(cfg, seed=0)
t = alto.AltoTensor.from_device_coo(cfg.dims, c, v); del c, v
R = cfg.rank
d = K.DeviceFactors([torch.rand((n, R), dtype=torch.float64, device="cuda") for n in cfg.dims], R)
p = MemoPlan(t, R, 0, 1)
o0 = torch.zeros((cfg.dims[0], nat.padded_ld(R)), dtype=torch.float64, device="cuda")
o1 = torch.zeros((cfg.dims[1], nat.padded_ld(R)), dtype=torch.float64, device="cuda")
for _ in range(3):
    p.mttkrp_m0(t, d, o0)
    p.mttkrp_m1(d, o1)
torch.cuda.synchronize()
print("ok", p.kind, p.P)
