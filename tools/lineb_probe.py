"""Time one level-2 line_b / line_b_const launch pair at N = 2^24 (5 components)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402
import torch  # noqa: E402
from paper_2411_09287_b200 import _lib  # noqa: E402

N, d, nc = 1 << 24, 64, 5
X = [torch.randint(-2**62, 2**62, (N,), dtype=torch.int64, device="cuda") for _ in range(nc)]
tabs = torch.randint(-2**62, 2**62, (4, N // 4, d), dtype=torch.int64, device="cuda")
g = torch.randint(-2**62, 2**62, (4, d), dtype=torch.int64, device="cuda")
outs = [torch.empty((N // 4, d), dtype=torch.int64, device="cuda") for _ in range(nc)]
P = C.c_void_p * 8
xc = P(*[x.data_ptr() for x in X], *([None] * (8 - nc)))
oc = P(*[o.data_ptr() for o in outs], *([None] * (8 - nc)))
m = (1 << 64) - 1


def lb():
    _lib.call("r3_vfy_line_b", 4, nc, xc, N, 1, 1, 1, tabs.data_ptr(), (N // 4) * d, 4, d, oc, m, _lib.stream())


def lbc():
    _lib.call("r3_vfy_line_b_const", 4, nc, xc, N, 1, 1, 1, g.data_ptr(), d, oc, m, _lib.stream())


for name, fn, gb in (("line_b", lb, (N * 8 * nc + N * 512 + nc * N // 4 * 512) / 1e9),
                     ("line_b_const", lbc, (N * 8 * nc + nc * N // 4 * 512) / 1e9)):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{name:14s} {ms:.3f} ms  {gb / ms:.0f} GB/s algorithmic")
