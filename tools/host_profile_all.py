"""cProfile of ALL threads (the coop engine runs each party on its own
thread) for one small mulv session; merged stats sorted by tottime and
cumulative.  Diagnostic only.

    python tools/host_profile_all.py [log2n]
"""
import cProfile
import os
import pstats
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2411_09287_b200 import verify  # noqa: E402
from paper_2411_09287_b200.runtime import Session  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 16
N = 1 << L
mulv, _ = bench.make_programs(N, 64, verify.pick_r(N, 64, 64))
for i in range(3):
    Session(seed=i).run(mulv)
torch.cuda.synchronize()

profiles = []
_orig_run = threading.Thread.run


def run(self):
    pr = cProfile.Profile()
    profiles.append(pr)
    pr.enable()
    try:
        _orig_run(self)
    finally:
        pr.disable()


threading.Thread.run = run
main = cProfile.Profile()
main.enable()
Session(seed=9).run(mulv)
torch.cuda.synchronize()
main.disable()
threading.Thread.run = _orig_run
st = pstats.Stats(main)
for p in profiles:
    st.add(p)
st.sort_stats("tottime").print_stats(30)
st.sort_stats("cumulative").print_stats(50)
