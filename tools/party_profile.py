"""cProfile of one party's thread (P1) over small sessions: the profiler is
enabled inside the party program, so only that thread is measured; time
parked on the coop baton shows up as lock acquires.

    python tools/party_profile.py [log2n] [role] [sessions]
"""
import cProfile
import os
import pstats
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2411_09287_b200 import verify  # noqa: E402
from paper_2411_09287_b200.runtime import Session  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 16
role = int(sys.argv[2]) if len(sys.argv) > 2 else 1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
N = 1 << L
prog, _ = bench.make_programs(N, 64, verify.pick_r(N, 64, 64))
pr = cProfile.Profile()


def wrapped(party):
    if party.role != role:
        return prog(party)
    pr.enable()
    try:
        return prog(party)
    finally:
        pr.disable()


for i in range(3):
    Session(seed=i).run(prog)
torch.cuda.synchronize()
for i in range(reps):
    Session(seed=10 + i).run(wrapped)
torch.cuda.synchronize()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(30)
st.sort_stats("cumulative").print_stats(45)
