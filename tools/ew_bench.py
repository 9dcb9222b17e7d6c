"""Achieved HBM bandwidth of the elementwise share kernels at 2^24 words."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2411_09287_b200 import _lib, grvec  # noqa: E402

n = 1 << 24
a = torch.randint(-2**62, 2**62, (n,), dtype=torch.int64, device="cuda")
b = torch.randint(-2**62, 2**62, (n,), dtype=torch.int64, device="cuda")
out = torch.empty_like(a)


def timeit(fn, nbytes, name):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"{name:28s} {ms * 1e3:8.1f} us  {nbytes / ms / 1e6:7.0f} GB/s")


timeit(lambda: _lib.call("r3_ew_flat", grvec.ADD, n, out.data_ptr(), a.data_ptr(), b.data_ptr(), 0,
                         (1 << 64) - 1, _lib.stream()), 3 * 8 * n, "ew_flat add")
timeit(lambda: grvec.ew_fields(grvec.ADD, [a, b], [b, a], (1 << 64) - 1), 6 * 8 * n, "ew_multi add x2")
timeit(lambda: torch.add(a, b, out=out), 3 * 8 * n, "torch add (reference)")
timeit(lambda: out.copy_(a), 2 * 8 * n, "torch copy (reference)")
