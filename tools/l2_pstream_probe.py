"""Streamed-Pi Phi throughput when Pi fits in L2 (small c4-distributed
tensors, Phi repeated back to back) vs the full c4 tensor: what an
L2-resident row-block CP-APR inner loop could gain."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic, kernels as K, _native as nat
from paper_2403_06348_b200.cpd import apr as A

cfg = synthetic.CONFIGS["c4"]
R = cfg.rank
for nnz in (250_000, 500_000, 1_000_000, 2_000_000, 50_000_000):
    c, v = synthetic.generate(cfg, seed=0, nnz=nnz)
    t = alto.AltoTensor.from_device_coo(cfg.dims, c, v); del c, v
    d = K.DeviceFactors([torch.rand((n, R), dtype=torch.float64, device="cuda") for n in cfg.dims], R)
    mode = 0
    A.prefer_unblocked(t, mode)
    b = torch.rand((cfg.dims[mode], nat.padded_ld(R)), dtype=torch.float64, device="cuda")
    out = torch.zeros_like(b)
    pil = torch.empty(A.pstream_sizes(t, R)[1], dtype=torch.float64, device="cuda")
    A.launch_phi(t, d, mode, "dview", b, 1e-10, out=out, pi_il_out=pil)
    f = lambda: A.launch_phi_pstream(t, mode, R, b, 1e-10, pil, out)
    f(); torch.cuda.synchronize()
    n = max(10, int(2e8 // nnz))
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    pib = pil.numel() * 8
    print(json.dumps({"nnz": t.nnz, "pi_MB": round(pib / 1e6, 1), "ms": round(ms, 4), "gnnz_s": round(t.nnz / ms / 1e6, 1),
                      "GBps_pi_stream": round((pib + t.nnz * 12) / ms / 1e6, 1), "reps": n}), flush=True)
    del t, pil, out, b, d; torch.cuda.empty_cache()
