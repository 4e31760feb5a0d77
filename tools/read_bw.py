"""Practical HBM read bandwidth on this GPU (calibration for the θ-pass roofline)."""
import torch

x = torch.randint(0, 1 << 30, (150_000_000,), dtype=torch.int32, device="cuda")
y = torch.empty_like(x)
ev = lambda: torch.cuda.Event(enable_timing=True)
for name, fn, nbytes in [("sum(int32) read-only", lambda: x.sum(), x.numel() * 4),
                         ("max(int32) read-only", lambda: x.max(), x.numel() * 4),
                         ("copy (read+write)", lambda: y.copy_(x), x.numel() * 8)]:
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = ev(), ev()
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    t = min(ts)
    print(f"{name}: {t*1e3:.1f} us  {nbytes/t/1e6:.0f} GB/s")
