"""How far the GPU lags behind the host protocol driver during one session
(honest coop engine, no per-call hooks): at every challenge opening of P0
the host time and a CUDA event are recorded; lag = (GPU time the event
completes) - (host time it was recorded).  Lag near zero means the GPU had
drained its queue there (host-bound stretch); a large lag means the host
ran ahead (GPU-bound).  Diagnostic only.

    python tools/host_gpu_lag.py 24 mulv
"""

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_09287_b200 import _lib, sharing, verify  # noqa: E402
from paper_2411_09287_b200.runtime import Session  # noqa: E402


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    what = sys.argv[2] if len(sys.argv) > 2 else "mulv"
    N = 1 << L
    if what == "mulv":
        prog, _ = bench.make_programs(N, 64, verify.pick_r(N, 64, 64))
        args = ()
    else:
        prog = bench.make_relu_program(N, 16)
        xv = np.trunc(np.random.default_rng(1).normal(0, 4, N) * 2 ** 16).astype(np.int64)
        args = (torch.from_numpy(xv).pin_memory(), True)
    for i in range(3):
        Session(seed=i).run(prog, *args)
    torch.cuda.synchronize()

    marks = []
    orig_rec = sharing.rec

    def rec(party, v, tag, *a, **k):
        out = orig_rec(party, v, tag, *a, **k)
        if party.role == 0:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            marks.append((tag, time.perf_counter(), e))
        return out

    last = [0.0]
    orig_call = _lib.call

    def call(name, *a):
        orig_call(name, *a)
        last[0] = time.perf_counter()

    sharing.rec = rec
    verify.rec = rec
    _lib.call = call
    for mod in list(sys.modules.values()):
        if getattr(mod, "__name__", "").startswith("paper_2411_09287_b200") and getattr(mod, "call", None) is orig_call:
            mod.call = call
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record()
    Session(seed=99).run(prog, *args)
    t_ret = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    t_end = time.perf_counter()
    gpu_total = e0.elapsed_time(e1)
    print(f"{what} 2^{L}: host last launch {1e3 * (last[0] - t0):.1f} ms, run() returned {1e3 * (t_ret - t0):.1f} ms, "
          f"GPU span {gpu_total:.1f} ms, drained {1e3 * (t_end - t0):.1f} ms, {len(marks)} marks")
    for tag, th, ev in marks:
        tg = e0.elapsed_time(ev)
        print(f"  {tag:14s} host {1e3 * (th - t0):7.2f}  gpu {tg:7.2f}  lag {tg - 1e3 * (th - t0):7.2f} ms")


if __name__ == "__main__":
    main()
