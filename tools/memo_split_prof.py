"""Time the memoised producer pieces on c2: fused memo0 vs split (sums + memo1 in T order)."""
import json, os, sys
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
def timed(f, n=10):
    f(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
for (m0, m1) in ((0, 1), (1, 2), (2, 0)):
    p = MemoPlan(t, R, m0, m1)
    out = torch.zeros((cfg.dims[m0], nat.padded_ld(R)), dtype=torch.float64, device="cuda")
    ak = d.mats[p.k]; a1 = d.mats[m1]
    sums = lambda: nat.call("alto_memo_sums", nat.ptr(p.pieceid), nat.ptr(p.crd[1 - p.jplane]), nat.ptr(p.vals), t.nnz,
                            nat.ptr(ak), ak.stride(0), R, nat.ptr(p.T), p.T.stride(0), nat.stream_ptr())
    cons_nat = lambda: nat.call("alto_mttkrp_memo1", nat.ptr(p.nrow), nat.ptr(p.ncrd), None, nat.ptr(p.T), p.T.stride(0),
                                p.P, nat.ptr(a1), a1.stride(0), R, nat.ptr(out), out.stride(0), nat.stream_ptr())
    p.split = False
    fused = lambda: p.mttkrp_m0(t, d, out)
    out1 = torch.zeros((cfg.dims[m1], nat.padded_ld(R)), dtype=torch.float64, device="cuda")
    cons = lambda: p.mttkrp_m1(d, out1)
    dv = lambda: K.launch_mttkrp(t, d, m0, "dview", out=out)
    print(json.dumps({"pair": [m0, m1], "P": p.P, "fused_ms": timed(fused), "sums_ms": timed(sums),
                      "memo1_T_order_ms": timed(cons_nat), "consumer_ms": timed(cons), "dview_ms": timed(dv)}), flush=True)
    del p; torch.cuda.empty_cache()
