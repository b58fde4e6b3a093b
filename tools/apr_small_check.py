"""c4 distribution at 2M nonzeros: GPU cp_apr_mu vs the oracle driver (log-likelihood traces incl. -inf)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic
from oracle import alto_oracle as orc
cfg = synthetic.CONFIGS["c4"]
c, v = synthetic.generate(cfg, seed=0, nnz=2_000_000)
hc, hv = c.cpu().numpy(), v.cpu().numpy()
t = alto.AltoTensor.from_device_coo(cfg.dims, c, v)
res = alto.cp_apr_mu(t, alto.CpAprConfig(rank=10, max_outer=5, max_inner=10, eps=1e-10, seed=0))
keys, sv, sc = orc.from_coo(cfg.dims, hc, hv)
th = len(os.sched_getaffinity(0))
w, fs, kk, inn, lls = orc.cp_apr(cfg.dims, sc, sv, 10, 5, max_inner=10, seed=0, eps=1e-10, strategy="recursive", L=th, threads=th, seg_cache={})
print("gpu", res.loglik_trace, res.inner_iters)
print("orc", lls, inn)
zero_rows = [int((f.sum(axis=1) == 0).sum()) for f in fs]
print("oracle all-zero factor rows per mode", zero_rows)
