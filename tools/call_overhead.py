"""Host cost of one tiny library call through the Python layers (no
protocol): raw ctypes call, grvec.add (allocates the output), torch.empty."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2411_09287_b200 import _lib, grvec  # noqa: E402

a = torch.zeros(64, dtype=torch.int64, device="cuda")
b = torch.zeros(64, dtype=torch.int64, device="cuda")
out = torch.empty(64, dtype=torch.int64, device="cuda")
n = 3000


def bench(name, fn):
    for _ in range(100):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    dt = (time.perf_counter() - t) / n
    torch.cuda.synchronize()
    print(f"{name:28s} {dt * 1e6:7.2f} us/call")


s = _lib.stream()
bench("torch.empty(64)", lambda: torch.empty(64, dtype=torch.int64, device="cuda"))
bench("_lib.stream()", lambda: _lib.stream())
bench("grvec.add (alloc + call)", lambda: grvec.add(a, b, 64))
bench("torch add", lambda: a + b)
