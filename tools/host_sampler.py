"""Sampling profile of the host protocol driver across ALL party threads
(cProfile only sees the thread that enabled it): a sampler thread reads
sys._current_frames() every ~200 us and charges each sample to the party
thread that is running (the one not parked on a coop lock), by innermost
package frame and by inclusive package function.  Diagnostic only.

    python tools/host_sampler.py mulv 20
"""

import collections
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_09287_b200 import verify  # noqa: E402
from paper_2411_09287_b200.runtime import Session  # noqa: E402

PKG = "paper_2411_09287_b200"


def main():
    kind, lg = sys.argv[1], int(sys.argv[2])
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
    N = 1 << lg
    if kind.startswith("relu"):
        rng = np.random.default_rng(1)
        xh = torch.from_numpy(np.trunc(rng.normal(0, 4, N) * 2 ** 16).astype(np.int64)).pin_memory()
        prog = bench.make_relu_program(N, 16)
        args = (xh, kind == "relu_v")
    else:
        prog, _ = bench.make_programs(N, 64, verify.pick_r(N, 64, 64))
        args = ()
    for i in range(3):
        Session(seed=i).run(prog, *args)
    torch.cuda.synchronize()
    sys.setswitchinterval(1e-4)
    inner = collections.Counter()
    incl = collections.Counter()
    lines = collections.Counter()
    stop = [False]
    n = [0]
    me = threading.get_ident()

    def sampler():
        while not stop[0]:
            time.sleep(2e-4)
            for tid, fr in sys._current_frames().items():
                if tid == me or tid == threading.get_ident():
                    continue
                # parked threads sit in lock.acquire inside runtime._Baton
                top = fr
                code = top.f_code
                if code.co_name in ("yield_to_scheduler", "resume", "_run_coop", "join", "wait"):
                    continue
                n[0] += 1
                seen = set()
                first = None
                f = fr
                while f is not None:
                    fn = f.f_code.co_filename
                    if PKG in fn or "bench.py" in fn:
                        key = f"{os.path.basename(fn)}:{f.f_code.co_name}"
                        if first is None:
                            first = key
                            lines[f"{os.path.basename(fn)}:{f.f_lineno}:{f.f_code.co_name}"] += 1
                        if key not in seen:
                            incl[key] += 1
                            seen.add(key)
                    f = f.f_back
                inner[first or f"<other>:{code.co_name}"] += 1

    th = threading.Thread(target=sampler, daemon=True)
    th.start()
    t0 = time.perf_counter()
    for i in range(reps):
        Session(seed=100 + i).run(prog, *args)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    stop[0] = True
    th.join()
    print(f"{kind} 2^{lg}: {reps} sessions, {1e3 * wall / reps:.1f} ms each, {n[0]} samples")
    tot = max(1, n[0])
    print("innermost package frame:")
    for k, v in inner.most_common(30):
        print(f"  {100 * v / tot:5.1f}%  {k}")
    print("inclusive:")
    for k, v in incl.most_common(40):
        print(f"  {100 * v / tot:5.1f}%  {k}")
    print("lines:")
    for k, v in lines.most_common(30):
        print(f"  {100 * v / tot:5.1f}%  {k}")


if __name__ == "__main__":
    main()
