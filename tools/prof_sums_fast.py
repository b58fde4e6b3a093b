"""Launch the branch-free piece-sum kernel on c2 pair (0, 1) a few times (for ncu)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic, kernels as K, _native as nat
os.environ["ALTO_B200_MEMO_SPLIT"] = "1"
from paper_2403_06348_b200.memo import MemoPlan
cfg = synthetic.CONFIGS["c2"]
c, v = synthetic.generate(cfg, seed=0)
t = alto.AltoTensor.from_device_coo(cfg.dims, c, v); del c, v
R = cfg.rank
d = K.DeviceFactors([torch.rand((n, R), dtype=torch.float64, device="cuda") for n in cfg.dims], R)
p = MemoPlan(t, R, 0, 1)
ak = d.mats[p.k]
n = ctypes.c_int64(0)
nat.call("alto_il_length", t.nnz, R, ctypes.byref(n))
kf = torch.empty(n.value, dtype=torch.int32, device="cuda")
fv = torch.empty(n.value, dtype=torch.float64, device="cuda")
nat.call("alto_memo_sums_stream", nat.ptr(p.rows), nat.ptr(p.crd[p.jplane]), nat.ptr(p.crd[1 - p.jplane]),
         nat.ptr(p.vals), t.nnz, R, nat.ptr(kf), nat.ptr(fv), nat.stream_ptr())
for _ in range(3):
    nat.call("alto_memo_sums_fast", nat.ptr(kf), nat.ptr(fv), t.nnz, nat.ptr(p.pbase), nat.ptr(ak), ak.stride(0), R,
             nat.ptr(p.T), p.T.stride(0), nat.stream_ptr())
torch.cuda.synchronize()
print("ok")
