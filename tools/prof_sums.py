"""c2: the memo piece-sum kernel (dview3<NO=1>) and the plain dview3 MTTKRP, two launches each (ncu target)."""
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
out = torch.zeros((cfg.dims[0], nat.padded_ld(R)), dtype=torch.float64, device="cuda")
K.launch_mttkrp(t, d, 0, "dview", out=out)
torch.cuda.synchronize()
ak = d.mats[p.k]
for _ in range(2):
    nat.call("alto_memo_sums", nat.ptr(p.pieceid), nat.ptr(p.crd[1 - p.jplane]), nat.ptr(p.vals), t.nnz,
             nat.ptr(ak), ak.stride(0), R, nat.ptr(p.T), p.T.stride(0), nat.stream_ptr())
for _ in range(2):
    K.launch_mttkrp(t, d, 0, "dview", out=out)
a1 = d.mats[1]
for _ in range(2):  # the producing mode's MTTKRP from T (pieces in T order)
    nat.call("alto_mttkrp_memo1", nat.ptr(p.nrow), nat.ptr(p.ncrd), None, nat.ptr(p.T), p.T.stride(0), p.P,
             nat.ptr(a1), a1.stride(0), R, nat.ptr(out), out.stride(0), nat.stream_ptr())
torch.cuda.synchronize()
print("ok")
