"""A few streamed-Pi Phi launches on a config (for ncu capture)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic, kernels as K
from paper_2403_06348_b200.cpd import apr as A
cfg = synthetic.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
c, v = synthetic.generate(cfg, seed=0)
t = alto.AltoTensor.from_device_coo(cfg.dims, c, v)
del c, v
R = cfg.rank
d = K.DeviceFactors([torch.rand((n, R), dtype=torch.float64, device="cuda") for n in cfg.dims], R)
pil = torch.empty(A.pstream_sizes(t, R)[1], dtype=torch.float64, device="cuda")
b = torch.rand((cfg.dims[0], K.nat.padded_ld(R)), dtype=torch.float64, device="cuda")
o = torch.zeros_like(b)
A.launch_phi(t, d, 0, "dview", b, 1e-10, out=o, pi_il_out=pil)
for _ in range(3):
    A.launch_phi_pstream(t, 0, R, b, 1e-10, pil, o)
torch.cuda.synchronize()
print("done")
