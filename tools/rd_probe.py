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
