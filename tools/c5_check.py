import os, sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic
from paper_2403_06348_b200.tensor import _strictly_increasing
cfg = synthetic.CONFIGS["c5"]
c, v = synthetic.generate(cfg, seed=0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
t = alto.AltoTensor.from_device_coo(cfg.dims, c, v)
e1.record(); torch.cuda.synchronize()
print("encode+sort ms", e0.elapsed_time(e1), "sorted", _strictly_increasing(t._keys), t._keys.shape, flush=True)
# unique coords check on a sample
u = torch.unique(c[:2000000], dim=0).shape[0]
print("sample unique", u)
