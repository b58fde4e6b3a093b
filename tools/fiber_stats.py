"""Mean nonzeros per (row, fiber-mode coordinate) fiber for every (mode,
fiber mode) pair of a synthetic config (chooses the fused kernel's fiber
mode). Usage: python tools/fiber_stats.py c5 [c3 ...]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2403_06348_b200 import synthetic

for name in sys.argv[1:]:
    cfg = synthetic.CONFIGS[name]
    coords, _vals = synthetic.generate(cfg, seed=0)
    del _vals
    M, N = coords.shape
    for m in range(N):
        for f in range(N):
            if f == m:
                continue
            key = coords[:, m] * cfg.dims[f] + coords[:, f]
            n = torch.unique(key).numel()
            del key
            torch.cuda.empty_cache()
            print(json.dumps({"cfg": name, "mode": m, "fiber_mode": f, "dims": [cfg.dims[m], cfg.dims[f]],
                              "fibers": n, "nnz_per_fiber": round(M / n, 3)}), flush=True)
    del coords
    torch.cuda.empty_cache()
