"""AES-128-CTR keystream kernel throughput (blocks/s) at bench sizes."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2411_09287_b200 import _lib  # noqa: E402
from paper_2411_09287_b200.prg import Prg  # noqa: E402

p = Prg(bytes(range(16)), "bench")
for n in (1 << 20, 1 << 24, 1 << 26):
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    f = lambda: _lib.call("r3_prf_ctr", p._rk, 12345, n, (1 << 64) - 1, 0, out.data_ptr(), _lib.stream())
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"prf_ctr n={n:>10d}: {ms:.3f} ms  {n / 2 / ms / 1e6:.2e} blocks/s  {8 * n / ms / 1e6:.0f} GB/s out")
lanes = 1 << 22
out = torch.empty(lanes, dtype=torch.int64, device="cuda")
f = lambda: _lib.call("r3_prf_bits_packed", p._rk, 0, 64, lanes, out.data_ptr(), _lib.stream())
f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
f()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"bits_packed 64 x {lanes}: {ms:.3f} ms  {64 * lanes / 2 / ms / 1e6:.2e} blocks/s")
