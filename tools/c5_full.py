"""c5 at full size on one GPU: lean generation, encode + sort, per-mode MTTKRP."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic, kernels as K
cfg = synthetic.CONFIGS["c5"]
torch.cuda.synchronize(); t0 = time.perf_counter()
c, v = synthetic.generate(cfg, seed=0)
torch.cuda.synchronize(); t1 = time.perf_counter()
t = alto.AltoTensor.from_device_coo(cfg.dims, c, v); del c, v
torch.cuda.synchronize(); t2 = time.perf_counter()
print("gen_s", round(t1 - t0, 2), "encode_sort_s", round(t2 - t1, 3), "nnz", t.nnz, "bits", t.layout.total_bits,
      "mem_GB", round(torch.cuda.max_memory_allocated() / 1e9, 1), flush=True)
R = cfg.rank
fac = K.DeviceFactors([torch.rand((d, R), dtype=torch.float64, device="cuda") for d in cfg.dims], R)
for n in range(5):
    kern, why = K.select_gpu_kernel(t, n, R, None)
    out = K.launch_mttkrp(t, fac, n, kern); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): K.launch_mttkrp(t, fac, n, kern, out=out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    B = synthetic.algorithmic_bytes(cfg, t.nnz, R, 16)
    print({"mode": n, "kernel": kern, "ms": round(ms, 2), "gnnz_s": round(t.nnz / ms / 1e6, 2),
           "frac": round(B / ms / 1e6 / 6539.2, 4), "mem_GB": round(torch.cuda.max_memory_allocated() / 1e9, 1)},
          flush=True)
    t._cache.clear(); torch.cuda.empty_cache()
