"""c3 mode 3 (168 rows, R = 32): dview3 vs the ALTO segment kernel, one launch each after a warm-up (ncu target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic, kernels as K
cfg = synthetic.CONFIGS["c3"]
c, v = synthetic.generate(cfg, seed=0)
t = alto.AltoTensor.from_device_coo(cfg.dims, c, v); del c, v
R = cfg.rank
d = K.DeviceFactors([torch.rand((n, R), dtype=torch.float64, device="cuda") for n in cfg.dims], R)
out = K.launch_mttkrp(t, d, 3, "dview")
K.launch_mttkrp(t, d, 3, "segment", out=out)
torch.cuda.synchronize()
K.launch_mttkrp(t, d, 3, "dview", out=out)
K.launch_mttkrp(t, d, 3, "segment", out=out)
torch.cuda.synchronize()
print("ok")
