"""Where the POST phase of one verified secure-ReLU session goes, per log
(mul.arith / dot.arith / mul.bool): wall time from the first party entering
a log's batch verification to the last one leaving it (coop engine, so the
three parties' work on that log is inside the window), device drained at
both ends, plus the GPU time of the library calls made inside it.
Diagnostic only.

    python tools/vfy_split.py 20
"""

import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_09287_b200 import _lib, verify  # noqa: E402
from paper_2411_09287_b200.runtime import Session  # noqa: E402


def main():
    log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    N = 1 << log2n
    prog = bench.make_relu_program(N, 16)
    xv = np.trunc(np.random.default_rng(1).normal(0, 4, N) * 2 ** 16).astype(np.int64)
    xh = torch.from_numpy(xv).pin_memory()
    for i in range(2):
        Session(seed=i).run(prog, xh, True)
    torch.cuda.synchronize()

    win = {}
    active = collections.Counter()
    cur = []
    gpu = collections.Counter()
    calls = collections.Counter()
    kern = collections.defaultdict(collections.Counter)

    def wrap(fn, tag):
        def inner(party, base_ell, *a, **k):
            key = f"{tag}.{'bool' if base_ell == 1 else 'arith'}"
            if active[key] == 0 and key not in win:
                torch.cuda.synchronize()
                win[key] = [time.perf_counter(), None]
            active[key] += 1
            cur.append(key)
            try:
                return fn(party, base_ell, *a, **k)
            finally:
                cur.remove(key)
                active[key] -= 1
                torch.cuda.synchronize()
                win[key][1] = time.perf_counter()
        return inner

    ev = []

    def hook(name, args, run):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        rc = run()
        e.record()
        ev.append((cur[-1] if cur else "other", name, s, e))
        return rc

    verify.batch_verify_muls = wrap(verify.batch_verify_muls, "mul")
    verify.batch_verify_dots = wrap(verify.batch_verify_dots, "dot")
    torch.cuda.reset_peak_memory_stats()
    w0 = time.perf_counter()
    _lib.CALL_HOOK = hook
    Session(seed=99).run(prog, xh, True)
    _lib.CALL_HOOK = None
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    for key, name, s, e in ev:
        t = s.elapsed_time(e)
        gpu[key] += t
        calls[key] += 1
        kern[key][name] += t
    print(f"relu 2^{log2n} verified session: wall {wall * 1e3:.1f} ms, peak {torch.cuda.max_memory_allocated() / 2**30:.1f} GiB")
    for key, (a, b) in win.items():
        print(f"  {key:10s} window {1e3 * (b - a):8.1f} ms  gpu {gpu[key]:8.1f} ms  calls {calls[key]}")
        for k, v in kern[key].most_common(6):
            print(f"      {k:28s} {v:8.2f} ms")
    print(f"  outside    gpu {gpu['other']:8.1f} ms  calls {calls['other']}")


if __name__ == "__main__":
    main()
