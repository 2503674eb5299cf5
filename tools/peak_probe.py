import torch, time
x = torch.empty(2_100_000_000 // 8, dtype=torch.int64, device="cuda").random_(0, 100)
y = torch.empty_like(x)
def t(f, reps=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
ms = t(lambda: x.sum()); print(f"read-only sum: {ms:.3f} ms = {x.numel()*8/ms/1e6:.0f} GB/s")
ms = t(lambda: y.copy_(x)); print(f"copy: {ms:.3f} ms = {2*x.numel()*8/ms/1e6:.0f} GB/s (r+w)")
xf = x.view(torch.float64)
ms = t(lambda: xf.amax()); print(f"amax f64: {ms:.3f} ms = {x.numel()*8/ms/1e6:.0f} GB/s")
