"""Host cost of the primitives the protocol driver repeats (one B200):
a ctypes call without CUDA work, a tiny kernel launch through the C ABI,
torch.empty / torch.zeros of small device tensors, the same launch
through a GIL-holding handle (ctypes.PyDLL).  Diagnostic only."""

import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2411_09287_b200 import _lib  # noqa: E402


def per_call(fn, n=20000):
    for _ in range(200):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return 1e6 * (t1 - t0) / n


def main():
    lib = _lib.load()
    a = torch.zeros(64, dtype=torch.int64, device="cuda")
    o = torch.empty_like(a)
    st = _lib.stream()
    pa, po = a.data_ptr(), o.data_ptr()
    py = C.PyDLL(_lib.LIB_PATH)
    for name, args in _lib._SIGS.items():
        f = getattr(py, name)
        f.argtypes = args
        f.restype = _lib._RESTYPE.get(name, C.c_int)
    rows = [
        ("ctypes r3_abi_version (no CUDA)", lambda: lib.r3_abi_version()),
        ("ctypes r3_ew_flat n=64 (launch)", lambda: lib.r3_ew_flat(0, 64, po, pa, pa, 0, (1 << 64) - 1, st)),
        ("PyDLL r3_ew_flat n=64 (launch, GIL held)", lambda: py.r3_ew_flat(0, 64, po, pa, pa, 0, (1 << 64) - 1, st)),
        ("_lib.call r3_ew_flat + stream()", lambda: _lib.call("r3_ew_flat", 0, 64, po, pa, pa, 0, (1 << 64) - 1,
                                                                 _lib.stream())),
        ("torch.empty((1, 64))", lambda: torch.empty((1, 64), dtype=torch.int64, device="cuda")),
        ("_lib.empty((1, 64))", lambda: _lib.empty((1, 64))),
        ("_lib.zeros((2, 127))", lambda: _lib.zeros((2, 127))),
        ("_lib.stream()", lambda: _lib.stream()),
        ("t.data_ptr()", lambda: a.data_ptr()),
        ("t[0:1] view", lambda: a[0:1]),
    ]
    for name, fn in rows:
        print(f"  {per_call(fn):7.2f} us  {name}")


if __name__ == "__main__":
    main()
