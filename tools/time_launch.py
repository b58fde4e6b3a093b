import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic, kernels as K
cfg = synthetic.CONFIGS["c2"]
coords, vals = synthetic.generate(cfg, seed=0, nnz=int(float(sys.argv[1])) if len(sys.argv) > 1 else cfg.nnz)
t = alto.AltoTensor.from_device_coo(cfg.dims, coords, vals); del coords
R = 16
fac = [torch.rand((d, R), dtype=torch.float64, device="cuda") for d in cfg.dims]
d = K.DeviceFactors(fac, R)
out = K.launch_mttkrp(t, d, 0, "oriented")
torch.cuda.synchronize()
for trial in range(3):
    t0 = time.perf_counter()
    K.launch_mttkrp(t, d, 0, "oriented", out=out)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"host enqueue {1e3*(t1-t0):.3f} ms, total {1e3*(t2-t0):.3f} ms", flush=True)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): K.launch_mttkrp(t, d, 0, "oriented", out=out)
e1.record(); torch.cuda.synchronize(); print("events per call ms", e0.elapsed_time(e1) / 10)
