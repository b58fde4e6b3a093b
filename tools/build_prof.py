"""Per-C-call device time of the layout builds (fused streams, memo plans) on a config."""
import collections, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic, partition, kernels as K, _native as nat
from paper_2403_06348_b200.memo import MemoPlan
cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = synthetic.CONFIGS[cfgname]
c, v = synthetic.generate(cfg, seed=0)
t = alto.AltoTensor.from_device_coo(cfg.dims, c, v); del c, v
R = cfg.rank
rec = []
orig = nat.call
def call(name, *a):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); orig(name, *a); e1.record(); rec.append((name, e0, e1))
nat.call = call
partition.nat.call = call
def report(tag, f):
    rec.clear(); torch.cuda.synchronize(); t0 = time.perf_counter()
    f(); torch.cuda.synchronize(); wall = (time.perf_counter() - t0) * 1e3
    agg = collections.OrderedDict()
    for n, a, b in rec: agg[n] = agg.get(n, 0.0) + a.elapsed_time(b)
    print(json.dumps({"cfg": cfgname, "what": tag, "wall_ms": round(wall, 2), "calls": {k: round(x, 3) for k, x in agg.items()}}), flush=True)
for rep in range(2):
    for m in range(len(cfg.dims)):
        t._cache.clear(); t._views.clear()
        fm = K._fused_fiber_mode(t, m)
        report(f"fused_stream mode {m} rep {rep}", lambda: partition.device_fused_stream(t, m, fm, R))
if len(cfg.dims) == 3:
    for m in range(3):
        t._cache.clear(); t._views.clear()
        report(f"memo plan {m}->{(m+1)%3}", lambda: MemoPlan(t, R, m, (m + 1) % 3))
