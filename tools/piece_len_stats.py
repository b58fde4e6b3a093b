"""Distribution of memo piece lengths (nonzeros per (i, j) piece of a
segment) on c2 for each pair."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic
from paper_2403_06348_b200.memo import MemoPlan
cfg = synthetic.CONFIGS["c2"]
c, v = synthetic.generate(cfg, seed=0)
t = alto.AltoTensor.from_device_coo(cfg.dims, c, v); del c, v
for m0, m1 in ((0, 1), (1, 2), (2, 0)):
    idx = MemoPlan._build_index(t, m0, m1)
    vals, rows, crd, pbase, prow, pcrd, pid, P = idx
    jp = m1 if m1 < m0 else m1 - 1
    M = t.nnz
    r = rows[:M].long(); j = crd[jp][:M].long()
    x = torch.arange(M, device="cuda")
    start = torch.ones(M, dtype=torch.bool, device="cuda")
    start[1:] = (r[1:] != r[:-1]) | (j[1:] != j[:-1])
    start |= (x % 512) == 0
    pos = torch.nonzero(start).flatten()
    lens = torch.diff(torch.cat([pos, torch.tensor([M], device="cuda")]))
    hist = {str(k): int((lens == k).sum()) for k in range(1, 6)}
    print(json.dumps({"pair": [m0, m1], "P": int(pos.numel()), "len_hist_1_5": hist,
                      "nnz_in_singletons": int((lens == 1).sum()), "mean_len": float(lens.float().mean())}), flush=True)
    del idx
