"""cProfile of a cold and a warm cp_als(c2, rank 16, 10 iterations): where the host time goes."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic
cfg = synthetic.CONFIGS["c2"]
c, v = synthetic.generate(cfg, seed=0)
t0 = alto.AltoTensor.from_device_coo(cfg.dims, c, v); del c, v
acfg = alto.CpAlsConfig(rank=16, max_iters=10, fit_tol=1e-300, seed=0)
def fresh(): return alto.AltoTensor(t0.layout, t0._keys, t0._vals, _validate=False)
alto.cp_als(fresh(), acfg)  # first-use costs (module load, attributes)
torch.cuda.synchronize(); torch.cuda.empty_cache()
for label in ("cold", "warm"):
    t = fresh() if label == "cold" else t
    torch.cuda.synchronize(); a = time.perf_counter()
    pr = cProfile.Profile(); pr.enable()
    alto.cp_als(t, acfg)
    pr.disable(); torch.cuda.synchronize()
    print(label, "s", time.perf_counter() - a, flush=True)
    pstats.Stats(pr).sort_stats("tottime").print_stats(14)
