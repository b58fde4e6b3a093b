"""A/B of the fiber-factored dview kernels (ALTO_B200_FIB) against dview3,
blocked and unblocked views: max relative difference and per-mode times.
python tools/fib_ab.py c2 mttkrp|phi"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic, kernels as K
from paper_2403_06348_b200.cpd import apr as A

cfgname, op = sys.argv[1], sys.argv[2]
variants = sys.argv[3].split(",") if len(sys.argv) > 3 else ["b1f0", "b1f1", "b0f0", "b0f1"]
cfg = synthetic.CONFIGS[cfgname]
coords, vals = synthetic.generate(cfg, seed=0)
t = alto.AltoTensor.from_device_coo(cfg.dims, coords, vals)
del coords, vals
R = cfg.rank
g = torch.Generator(device="cuda").manual_seed(0)
fac = [torch.rand((d, R), dtype=torch.float64, device="cuda", generator=g) for d in cfg.dims]
d = K.DeviceFactors(fac, R)
bs = [torch.rand((dm, K.nat.padded_ld(R)), dtype=torch.float64, device="cuda", generator=g) for dm in cfg.dims]
W = 8 if t.layout.word_bits == 64 else 16
ref = {}
tot = {}
for var in variants:
    blk, fib = var[1], var[3]
    os.environ["ALTO_B200_BLOCK"] = blk
    os.environ["ALTO_B200_FIB"] = "1" if fib == "1" else "0"
    os.environ["ALTO_B200_FIBER_ORDER"] = "long" if var.endswith("L") else "short"
    t._cache.clear()
    torch.cuda.empty_cache()
    tot[var] = 0.0
    for mode in range(len(cfg.dims)):
        if op == "mttkrp":
            f = lambda out=None: K.launch_mttkrp(t, d, mode, "dview", out=out)
        else:
            f = lambda out=None: A.launch_phi(t, d, mode, "dview", bs[mode], 1e-10, out=out)
        out = f(); torch.cuda.synchronize()
        o = out[:, :R].clone()
        if mode not in ref:
            ref[mode] = o
            err = 0.0
        else:
            err = float(((o - ref[mode]).abs() / ref[mode].abs().clamp_min(1e-300)).max())
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): f(out)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        tot[var] += ms
        print(json.dumps({"cfg": cfgname, "op": op, "var": var, "mode": mode, "ms": round(ms, 4),
                          "gnnz_s": round(t.nnz / ms / 1e6, 2), "max_rel_vs_first": err}), flush=True)
    print(json.dumps({"cfg": cfgname, "op": op, "var": var, "sum_ms": round(tot[var], 3)}), flush=True)
