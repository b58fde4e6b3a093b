"""Encoder timing on c2: linearise + radix sort of (key, value), device events."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic
cfg = synthetic.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
c, v = synthetic.generate(cfg, seed=0)
for rep in range(4):
    cc, vv = c.clone(), v.clone()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if rep == 3: torch.cuda.nvtx.range_push("enc")
    e0.record()
    t = alto.AltoTensor.from_device_coo(cfg.dims, cc, vv)
    e1.record(); torch.cuda.synchronize()
    if rep == 3: torch.cuda.nvtx.range_pop()
    print(cfg.name, "encode+sort ms", round(e0.elapsed_time(e1), 3), "nnz", t.nnz, flush=True)
    del t, cc, vv
