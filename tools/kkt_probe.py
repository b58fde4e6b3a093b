import sys; sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
import paper_2403_06348_b200 as alto
from conftest import random_sparse
from paper_2403_06348_b200.cpd import apr as APR
rng = np.random.default_rng(12)
coords, vals = random_sparse(rng, (60, 45, 70), 6000, kind="counts")
t = alto.AltoTensor.from_coo(alto.CooTensor((60, 45, 70), coords, vals))
st = APR.AprState(t, alto.CpAprConfig(rank=4, max_outer=4, max_inner=10, seed=3, tau=1e-4))
for _ in range(4): st.outer()
print("kkt", st.kkt_trace); print("inner", st.inner_counts)
