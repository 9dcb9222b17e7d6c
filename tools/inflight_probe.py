"""Throughput of verified-multiplication sessions run one at a time vs two
in flight (two host threads, one GPU, same stream): how much device time a
single session leaves idle while its host-bound verification tail runs.

    python tools/inflight_probe.py [log2n] [sessions]
"""
import os
import sys
import threading
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2411_09287_b200 import verify  # noqa: E402
from paper_2411_09287_b200.runtime import Session  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 24
S = int(sys.argv[2]) if len(sys.argv) > 2 else 6
N = 1 << L
prog, _ = bench.make_programs(N, 64, verify.pick_r(N, 64, 64))
for i in range(2):
    Session(seed=i).run(prog)
torch.cuda.synchronize()

t0 = time.perf_counter()
for i in range(S):
    assert all(Session(seed=10 + i).run(prog))
torch.cuda.synchronize()
seq = time.perf_counter() - t0


def worker(k):
    torch.cuda.set_device(0)
    for i in range(k, S, 2):
        assert all(Session(seed=10 + i).run(prog))


t0 = time.perf_counter()
ths = [threading.Thread(target=worker, args=(k,)) for k in range(2)]
for t in ths:
    t.start()
for t in ths:
    t.join()
torch.cuda.synchronize()
par = time.perf_counter() - t0
print(f"N=2^{L}: sequential {S * N / seq:.3e} mults/s ({seq / S * 1e3:.1f} ms/session), "
      f"two in flight {S * N / par:.3e} mults/s ({par / S * 1e3:.1f} ms/session)")
