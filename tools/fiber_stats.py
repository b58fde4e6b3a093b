"""Unique (row, other-mode) pairs per mode for a config: average fiber length
= M / pairs (how many gathers a fiber-factored kernel would save)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2403_06348_b200 import synthetic
cfg = synthetic.CONFIGS[sys.argv[1]]
c, v = synthetic.generate(cfg, seed=0)
M = c.shape[0]
N = len(cfg.dims)
for n in range(N):
    for m in range(N):
        if m == n:
            continue
        key = c[:, n].to(torch.int64) * cfg.dims[m] + c[:, m].to(torch.int64)
        u = torch.unique(key).numel()
        print(f"mode {n} x {m}: pairs {u}, avg fiber {M / u:.2f}", flush=True)
