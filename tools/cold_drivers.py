"""Cold public drivers on the BASELINE configs (for an ncu launch list): cp_als(c2, 10 iterations) and
cp_apr_mu(c4, 5 x 10), layouts built inside the calls."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic
which = sys.argv[1] if len(sys.argv) > 1 else "both"
if which in ("als", "both"):
    cfg = synthetic.CONFIGS["c2"]
    c, v = synthetic.generate(cfg, seed=0)
    t = alto.AltoTensor.from_device_coo(cfg.dims, c, v); del c, v
    torch.cuda.synchronize(); t0 = time.perf_counter()
    torch.cuda.nvtx.range_push("cp_als_cold")
    r = alto.cp_als(t, alto.CpAlsConfig(rank=16, max_iters=10, fit_tol=1e-300, seed=0))
    torch.cuda.synchronize(); torch.cuda.nvtx.range_pop()
    print("cp_als cold s", time.perf_counter() - t0, r.fit_trace[-1], flush=True)
    del t
if which in ("apr", "both"):
    cfg = synthetic.CONFIGS["c4"]
    c, v = synthetic.generate(cfg, seed=0)
    t = alto.AltoTensor.from_device_coo(cfg.dims, c, v); del c, v
    torch.cuda.synchronize(); t0 = time.perf_counter()
    torch.cuda.nvtx.range_push("cp_apr_cold")
    r = alto.cp_apr_mu(t, alto.CpAprConfig(rank=10, max_outer=5, max_inner=10, eps=1e-10, seed=0))
    torch.cuda.synchronize(); torch.cuda.nvtx.range_pop()
    print("cp_apr cold s", time.perf_counter() - t0, r.loglik_trace[-1], flush=True)
