"""Where the host time of one small session goes (single process, coop
engine): time inside library calls (ctypes + launch), device allocations,
coop yields (parked time while other parties run is excluded by measuring
wall time per party slice), message send/recv bookkeeping.

    python tools/host_split.py [log2n] [mulv|relu]
"""
import collections
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2411_09287_b200 import _lib, verify, runtime, transport  # noqa: E402
from paper_2411_09287_b200.runtime import Session  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 16
what = sys.argv[2] if len(sys.argv) > 2 else "mulv"
N = 1 << L
if what == "mulv":
    prog, _ = bench.make_programs(N, 64, verify.pick_r(N, 64, 64))
    args = ()
else:
    prog = bench.make_relu_program(N, 16)
    xv = np.trunc(np.random.default_rng(1).normal(0, 4, N) * 2 ** 16).astype(np.int64)
    args = (torch.from_numpy(xv), True)
for i in range(3):
    Session(seed=i).run(prog, *args)
torch.cuda.synchronize()

acc = collections.Counter()
cnt = collections.Counter()


def timed(name, fn):
    def w(*a, **k):
        t = time.perf_counter()
        try:
            return fn(*a, **k)
        finally:
            acc[name] += time.perf_counter() - t
            cnt[name] += 1
    return w


_lib.call = timed("lib.call", _lib.call)
for mod in list(sys.modules.values()):
    if mod and getattr(mod, "__name__", "").startswith("paper_2411_09287_b200") and hasattr(mod, "call"):
        if getattr(mod, "call") is not _lib.call:
            mod.call = _lib.call
_lib.empty = timed("lib.empty", _lib.empty)
for mod in list(sys.modules.values()):
    if mod and getattr(mod, "__name__", "").startswith("paper_2411_09287_b200") and hasattr(mod, "empty"):
        mod.empty = _lib.empty
b = runtime._Baton
b.yield_to_scheduler = timed("coop.yield(parked)", b.yield_to_scheduler)
transport.CoopRouter.send = timed("router.send", transport.CoopRouter.send)
Session._settle_deferred = timed("settle (device drain)", Session._settle_deferred)
import torch as _t  # noqa: E402
_t.Tensor.item = timed("tensor.item (sync)", _t.Tensor.item)

t0 = time.perf_counter()
Session(seed=9).run(prog, *args)
torch.cuda.synchronize()
tot = time.perf_counter() - t0
print(f"{what} 2^{L}: session {tot * 1e3:.1f} ms")
for k, v in acc.most_common():
    print(f"  {k:22s} {v * 1e3:8.2f} ms  n={cnt[k]}")
