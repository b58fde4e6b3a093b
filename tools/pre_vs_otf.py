"""Phi on c4: OTF (gathers) vs PRE (Khatri-Rao rows precomputed in view order)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic, kernels as K
from paper_2403_06348_b200.cpd import apr as A
from paper_2403_06348_b200.partition import dview_order
cfg = synthetic.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
c, v = synthetic.generate(cfg, seed=0)
t = alto.AltoTensor.from_device_coo(cfg.dims, c, v); del c, v
R = cfg.rank
fac = [torch.rand((d, R), dtype=torch.float64, device="cuda") for d in cfg.dims]
d = K.DeviceFactors(fac, R)
def ev(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for mode in range(3):
    b = torch.rand((cfg.dims[mode], K.nat.padded_ld(R)), dtype=torch.float64, device="cuda")
    out = torch.zeros_like(b)
    otf = ev(lambda: A.launch_phi(t, d, mode, "dview", b, 1e-10, out=out))
    keys = dview_order(t, mode, R)[1]
    pi = A.launch_pi_dview(t, d, mode)
    build = ev(lambda: A.launch_pi_dview(t, d, mode), reps=2)
    pre = ev(lambda: A.launch_phi(t, d, mode, "dview", b, 1e-10, pi_view=pi, out=out))
    print({"mode": mode, "otf_ms": round(otf, 3), "pre_ms": round(pre, 3), "pi_build_ms": round(build, 3),
           "pi_GB": round(pi.numel() * 8 / 1e9, 2)}, flush=True)
    del pi
