"""Small inputs through every kernel family, for compute-sanitizer runs
(memcheck / racecheck / synccheck, one tool per run): encoder (encode, radix
sort, canonicalisation with duplicates and cancellations), partition, every
MTTKRP / Phi kernel, the memoised CP-ALS sweep, CP-APR with the streamed-Pi
inner loop, the ALTO segment kernel and the deterministic mode."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import kernels as K
from paper_2403_06348_b200.cpd import apr as A

rng = np.random.default_rng(0)
# worked example (pkg/tests worked example shape)
t0 = alto.AltoTensor.from_coo(alto.CooTensor((4, 8, 2), [[0, 3, 0], [1, 0, 0], [1, 6, 1], [2, 2, 1], [3, 1, 1], [3, 4, 0]],
                                             [1.0, 2.0, 3.0, 4.0, 5.0, 6.0]))
# random tensor with duplicates and exact cancellations
dims = (37, 23, 41)
c = rng.integers(0, 23, (5000, 3)) % np.array(dims)
v = rng.random(5000) + 0.05
c = np.concatenate([c, c[:50]]); v = np.concatenate([v, -v[:50]])
t = alto.AltoTensor.from_coo(alto.CooTensor(dims, c, v))
for tt, R in ((t0, 3), (t, 16), (t, 5)):
    fac = [rng.random((d, R)) for d in tt.shape.dims]
    d = K.DeviceFactors(fac, R)
    for mode in range(3):
        for kern in ("dview", "oriented", "atomic", "segment", "segment-atomic", "exact-seq", "exact-rec", "exact-output"):
            K.launch_mttkrp(tt, d, mode, kern, num_segments=3)
        b = K.nat.to_device_matrix(rng.random((tt.shape.dims[mode], R)) + 0.1)
        for kern in ("dview", "oriented", "atomic"):
            A.launch_phi(tt, d, mode, kern, b, 1e-10)
    alto.make_segments(tt, 4).boundary_rows
alto.cp_als(t, alto.CpAlsConfig(rank=8, max_iters=3, fit_tol=1e-300))
cnt = alto.AltoTensor.from_coo(alto.CooTensor(dims, c[:5000], np.floor(v[:5000] * 5) + 1.0))
alto.cp_apr_mu(cnt, alto.CpAprConfig(rank=4, max_outer=3, max_inner=4))
alto.set_deterministic(True)
t2 = alto.AltoTensor(t.layout, t._keys, t._vals, _validate=False)
alto.cp_als(t2, alto.CpAlsConfig(rank=8, max_iters=2, fit_tol=1e-300))
alto.set_deterministic(False)
torch.cuda.synchronize()
print("sanitize case ok")
