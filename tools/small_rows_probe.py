"""Latency of one line evaluation (rows . M(1-z) + rows' . M(z), d = 64 / 16)
at small row counts: tensor-core kernel vs the CUDA-core matrix kernel.
Each launch timed alone (synchronised before, CUDA events around it)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2411_09287_b200 import grvec, _lib
from paper_2411_09287_b200.rings import modulus_for_degree

def t_one(fn, reps=30):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)

for d in (64, 16):
    mod = modulus_for_degree(d)
    rng = np.random.default_rng(0)
    z = grvec.dev(rng.integers(0, 2**63, (1, d), dtype=np.int64).view(np.uint64))
    one_m = grvec.sub(grvec.gr_const(1, mod, 64), z, 64)
    M0, M1 = grvec.gr_mulmat(one_m, mod), grvec.gr_mulmat(z, mod)
    for rows in (1, 8, 64, 128, 512, 2048, 8192, 32768, 131072):
        X = grvec.dev(rng.integers(0, 2**63, (2 * rows, d), dtype=np.int64).view(np.uint64))
        ev, od = X[0::2], X[1::2]
        tc = t_one(lambda: grvec.rows_times(ev, M0, rows, 64, P1=od, M1=M1))
        cc = t_one(lambda: grvec.gr_matmul(grvec.lin((1, od), (-1, ev)), M1, rows, d, 64, C_add=grvec.lin((1, ev))))
        a = grvec.rows_times(ev, M0, rows, 64, P1=od, M1=M1)
        b = grvec.gr_matmul(grvec.lin((1, od), (-1, ev)), M1, rows, d, 64, C_add=grvec.lin((1, ev)))
        assert torch.equal(a, b)
        print(f"d={d} rows={rows:7d}  tc {tc:8.1f} us   cuda-core {cc:8.1f} us", flush=True)
