"""Kernel-only timing of MTTKRP/Phi per mode on a synthetic config."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic, kernels as K
from paper_2403_06348_b200.cpd import apr as A
cfgname = sys.argv[1]; kernels = sys.argv[2].split(","); ops = sys.argv[3].split(",") if len(sys.argv) > 3 else ["mttkrp"]
cfg = synthetic.CONFIGS[cfgname]
coords, vals = synthetic.generate(cfg, seed=0)
t = alto.AltoTensor.from_device_coo(cfg.dims, coords, vals); del coords
R = cfg.rank
fac = [torch.rand((d, R), dtype=torch.float64, device="cuda") for d in cfg.dims]
d = K.DeviceFactors(fac, R)
W = 8 if t.layout.word_bits == 64 else 16
lib = os.environ.get("ALTO_B200_LIB", "default")
for op in ops:
  for kern in kernels:
    tot = 0.0
    for mode in range(len(cfg.dims)):
        if op == "mttkrp":
            f = lambda out=None: K.launch_mttkrp(t, d, mode, kern, out=out)
            B = synthetic.algorithmic_bytes(cfg, t.nnz, R, W)
        else:
            b = torch.rand((cfg.dims[mode], K.nat.padded_ld(R)), dtype=torch.float64, device="cuda")
            f = lambda out=None: A.launch_phi(t, d, mode, kern, b, 1e-10, out=out)
            B = synthetic.algorithmic_bytes(cfg, t.nnz, R, W, "phi", mode)
        try:
            out = f(); torch.cuda.synchronize()
        except Exception as ex:
            print(json.dumps({"cfg": cfgname, "op": op, "kernel": kern, "mode": mode, "error": str(ex)[:200]}), flush=True)
            t._cache.clear(); t._views.clear(); torch.cuda.empty_cache()
            continue
        extra = {}
        if kern.startswith("segment"):
            pl = K.segment_plan(t, mode, R)
            extra = {"L": pl["L"], "acc_rows": pl["acc_rows"], "mean_width": round(pl["mean_width"], 1),
                     "smem": pl["smem_bytes"]}
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): f(out)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5; tot += ms
        del out
        t._cache.clear(); t._views.clear(); torch.cuda.empty_cache()
        print(json.dumps({"lib": os.path.basename(lib), "cfg": cfgname, "op": op, "kernel": kern, "mode": mode, "ms": round(ms, 4),
                          "gnnz_s": round(t.nnz / ms / 1e6, 2), "frac": round(B / ms / 1e6 / 6539.2, 4), **extra}), flush=True)
    print(json.dumps({"lib": os.path.basename(lib), "cfg": cfgname, "op": op, "kernel": kern, "sum_ms": round(tot, 3)}), flush=True)
