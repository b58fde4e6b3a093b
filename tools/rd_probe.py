import torch
x = torch.rand(575_000_000, dtype=torch.float64, device="cuda")  # 4.6 GB
def ev(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
ms = ev(lambda: x.sum())
print("sum ms", ms, "GB/s", 4.6e9 / ms / 1e6)
y = torch.empty_like(x)
ms = ev(lambda: y.copy_(x))
print("copy ms", ms, "GB/s (r+w)", 9.2e9 / ms / 1e6)
# host <-> device (pinned) bandwidth: the floor of the public-API e2e
h = torch.empty(12_500_000 // 8, dtype=torch.float64, pin_memory=True)
dd = torch.empty_like(h, device="cuda")
ms = ev(lambda: dd.copy_(h, non_blocking=True))
print("H2D pinned 12.5 MB ms", ms, "GB/s", 12.5e6 / ms / 1e6)
h2 = torch.empty(6_300_000 // 8, dtype=torch.float64, pin_memory=True)
d2 = torch.empty_like(h2, device="cuda")
ms = ev(lambda: h2.copy_(d2, non_blocking=True))
print("D2H pinned 6.3 MB ms", ms, "GB/s", 6.3e6 / ms / 1e6)
