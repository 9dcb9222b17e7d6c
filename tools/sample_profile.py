"""Sampling profiler over all threads for small sessions (the coop engine
runs the parties on their own threads): every 100 us the stacks of every
thread are sampled; samples whose innermost package frame is a function are
counted (self) and every package frame on the stack is counted (inclusive).
Parked parties (waiting on the baton) are skipped.

    python tools/sample_profile.py [log2n] [mulv|relu] [sessions]
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

L = int(sys.argv[1]) if len(sys.argv) > 1 else 16
what = sys.argv[2] if len(sys.argv) > 2 else "mulv"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
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

PKG = "paper_2411_09287_b200"
self_c, incl_c = collections.Counter(), collections.Counter()
stop = False
me = threading.get_ident()


def sampler():
    while not stop:
        for tid, fr in sys._current_frames().items():
            if tid == me or tid == threading.get_ident():
                continue
            names = []
            f = fr
            parked = False
            while f is not None:
                co = f.f_code
                if co.co_name in ("yield_to_scheduler", "resume") and "runtime" in co.co_filename:
                    parked = True
                    break
                if PKG in co.co_filename or "bench.py" in co.co_filename:
                    names.append(f"{os.path.basename(co.co_filename)}:{co.co_name}")
                f = f.f_back
            if parked or not names:
                continue
            self_c[names[0]] += 1
            for n in set(names):
                incl_c[n] += 1
        time.sleep(0.0001)


th = threading.Thread(target=sampler, daemon=True)
th.start()
t0 = time.perf_counter()
for i in range(reps):
    Session(seed=10 + i).run(prog, *args)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
stop = True
th.join()
tot = sum(self_c.values())
print(f"{what} 2^{L}: {dt / reps * 1e3:.1f} ms/session, {tot} samples")
print("self:")
for k, v in self_c.most_common(25):
    print(f"  {100 * v / tot:5.1f}%  {k}")
print("inclusive:")
for k, v in incl_c.most_common(40):
    print(f"  {100 * v / tot:5.1f}%  {k}")
