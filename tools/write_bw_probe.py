"""Pure-write vs copy HBM bandwidth (torch fill / copy of 8 GB) for the roofline of write-heavy kernels."""
import torch
x = torch.empty(1 << 30, dtype=torch.int64, device="cuda")  # 8 GB
y = torch.empty(1 << 29, dtype=torch.int64, device="cuda")
for name, fn, gb in (("fill 8GB", lambda: x.fill_(3), 8.59), ("copy 4GB->4GB", lambda: x[: 1 << 29].copy_(y), 8.59)):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(name, f"{ms:.3f} ms", f"{gb / ms:.2f} TB/s")
