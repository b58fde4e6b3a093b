"""Scratch performance exploration on one GPU (not a bench)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic, kernels as K
from paper_2403_06348_b200.cpd import apr as A

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = synthetic.CONFIGS[cfgname]
nnz = int(float(sys.argv[2])) if len(sys.argv) > 2 else cfg.nnz
torch.cuda.synchronize()
t0 = time.perf_counter()
coords, vals = synthetic.generate(cfg, seed=0, nnz=nnz)
torch.cuda.synchronize(); t1 = time.perf_counter()
t = alto.AltoTensor.from_device_coo(cfg.dims, coords, vals)
torch.cuda.synchronize(); t2 = time.perf_counter()
print(json.dumps({"cfg": cfgname, "nnz": t.nnz, "gen_s": t1 - t0, "encode_sort_s": t2 - t1}), flush=True)
del coords
R = cfg.rank
fac = [torch.rand((d, R), dtype=torch.float64, device="cuda") for d in cfg.dims]
dfac = K.DeviceFactors(fac, R)
W = 8 if t.layout.word_bits == 64 else 16
B = synthetic.algorithmic_bytes(cfg, t.nnz, R, W)
res = {}
for kern in ("oriented", "atomic", "exact-output"):
    for mode in range(len(cfg.dims)):
        if kern == "exact-output" and mode > 0: continue
        out = K.launch_mttkrp(t, dfac, mode, kern, num_segments=K.nat.default_segments(t.nnz))
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record()
        for _ in range(reps):
            K.launch_mttkrp(t, dfac, mode, kern, out=out, num_segments=K.nat.default_segments(t.nnz))
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res[f"{kern}_m{mode}"] = ms
        print(json.dumps({"kernel": kern, "mode": mode, "ms": round(ms, 4), "gnnz_s": round(t.nnz / ms / 1e6, 2),
                          "GBs_alg": round(B / ms / 1e6, 1), "frac": round(B / ms / 1e6 / 6539.2, 4)}), flush=True)
# view build time
torch.cuda.synchronize(); t3 = time.perf_counter()
t._cache.clear(); 
from paper_2403_06348_b200.partition import device_mode_view
for m in range(len(cfg.dims)): device_mode_view(t, m)
torch.cuda.synchronize(); print(json.dumps({"view_build_s_all_modes": time.perf_counter() - t3}), flush=True)
if cfgname == "c4" or "--phi" in sys.argv:
    for kern in ("oriented", "atomic"):
        for mode in range(len(cfg.dims)):
            b = torch.rand((cfg.dims[mode], K.nat.padded_ld(R)), dtype=torch.float64, device="cuda")
            out = A.launch_phi(t, dfac, mode, kern, b, 1e-10)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5): A.launch_phi(t, dfac, mode, kern, b, 1e-10, out=out)
            e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1) / 5
            Bp = synthetic.algorithmic_bytes(cfg, t.nnz, R, W, "phi", mode)
            print(json.dumps({"phi": kern, "mode": mode, "ms": round(ms, 4), "frac": round(Bp / ms / 1e6 / 6539.2, 4)}), flush=True)
