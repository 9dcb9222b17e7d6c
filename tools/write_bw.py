"""HBM bandwidth of write-dominated traffic on this GPU (diagnostic for the
table kernel, which writes 4 bytes per byte it reads): torch fill (write
only) and copy (read + write) of 4 GiB, CUDA events, median of 5."""
import torch
n = 1 << 29  # 4 GiB of int64
a = torch.empty(n, dtype=torch.int64, device="cuda")
b = torch.empty(n, dtype=torch.int64, device="cuda")
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return sorted(ts)[len(ts) // 2]
s = t(lambda: a.fill_(7))
print(f"fill  {8 * n / s / 1e9:8.0f} GB/s (write only)")
s = t(lambda: b.copy_(a))
print(f"copy  {16 * n / s / 1e9:8.0f} GB/s (read + write)")
