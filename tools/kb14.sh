grep -h '"mode"\|sum_ms' gpurun_out/kb14.log
python - <<'PY' > gpurun_out/kb14.log 2>&1
import sys, time, torch
sys.path.insert(0, ".")
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic, kernels as K
cfg = synthetic.CONFIGS["c5"]
torch.cuda.synchronize(); t0 = time.perf_counter()
c, v = synthetic.generate(cfg, seed=0, nnz=62_500_000)  # one of 8 shards
torch.cuda.synchronize(); t1 = time.perf_counter()
t = alto.AltoTensor.from_device_coo(cfg.dims, c, v); del c, v
torch.cuda.synchronize(); t2 = time.perf_counter()
print("c5 gen", t1 - t0, "encode+sort", t2 - t1, "nnz", t.nnz, "bits", t.layout.total_bits, flush=True)
R = cfg.rank
fac = [torch.rand((d, R), dtype=torch.float64, device="cuda") for d in cfg.dims]
d = K.DeviceFactors(fac, R)
tot = 0
for mode in range(5):
    kern = K.select_gpu_kernel(t, mode, R, None)[0]
    out = K.launch_mttkrp(t, d, mode, kern); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): K.launch_mttkrp(t, d, mode, kern, out=out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3; tot += ms
    B = synthetic.algorithmic_bytes(cfg, t.nnz, R, 16)
    print({"cfg": "c5", "mode": mode, "kernel": kern, "ms": round(ms, 3), "frac": round(B / ms / 1e6 / 6539.2, 4)}, flush=True)
print("c5 sum_ms", tot, "mem GB", torch.cuda.max_memory_allocated() / 1e9)
PY
tail -8 gpurun_out/kb14.log
