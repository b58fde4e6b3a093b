"""Streamed-Pi Phi vs the gathering Phi on a config (default c4): per-mode
kernel times, agreement, and CP-APR seconds per outer iteration with
ALTO_B200_PSTREAM=0/1 (graph replays after three warm-up outers)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic, kernels as K
from paper_2403_06348_b200.cpd import apr as A

cfg = synthetic.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
c, v = synthetic.generate(cfg, seed=0)
t = alto.AltoTensor.from_device_coo(cfg.dims, c, v)
del c, v
R = cfg.rank
g = torch.Generator(device="cuda").manual_seed(0)
d = K.DeviceFactors([torch.rand((n, R), dtype=torch.float64, device="cuda", generator=g) for n in cfg.dims], R)


def ev(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


slots, pid = A.pstream_sizes(t, R)
pil = torch.empty(pid, dtype=torch.float64, device="cuda")
for mode in range(len(cfg.dims)):
    b = torch.rand((cfg.dims[mode], K.nat.padded_ld(R)), dtype=torch.float64, device="cuda", generator=g)
    o1 = torch.zeros_like(b); o2 = torch.zeros_like(b)
    otf = ev(lambda: A.launch_phi(t, d, mode, "dview", b, 1e-10, out=o1))
    wr = ev(lambda: A.launch_phi(t, d, mode, "dview", b, 1e-10, out=o1, pi_il_out=pil))
    ps = ev(lambda: A.launch_phi_pstream(t, mode, R, b, 1e-10, pil, o2))
    rel = float(((o2 - o1).abs().max() / o1.abs().max()))
    pre_bytes = t.nnz * (16 + 8 * R) + 16 * cfg.dims[mode] * R
    print(json.dumps({"lib": os.path.basename(os.environ.get("ALTO_B200_LIB", "default")), "mode": mode, "otf_ms": round(otf, 4), "otf_write_ms": round(wr, 4), "pstream_ms": round(ps, 4),
                      "max_rel": rel, "pstream_frac": round(pre_bytes / ps / 1e6 / 6539.2, 3)}), flush=True)
del pil
torch.cuda.empty_cache()

for flag in (() if os.environ.get("PS_NO_APR") else ("0", "1")):
    os.environ["ALTO_B200_PSTREAM"] = flag
    st = A.AprState(t, alto.CpAprConfig(rank=R, max_outer=5, max_inner=10, eps=1e-10, seed=0))
    for _ in range(3):
        st.outer()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        st.outer()
    e1.record(); torch.cuda.synchronize()
    print(json.dumps({"pstream": flag, "s_per_outer": e0.elapsed_time(e1) / 3e3, "inner": st.inner_counts[-1],
                      "loglik": st.loglik_trace[-1]}), flush=True)
    del st
    torch.cuda.empty_cache()
