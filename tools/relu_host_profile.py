"""cProfile of each party thread of one verified-ReLU session (diagnostic).
    python tools/relu_host_profile.py [log2n]"""
import cProfile
import io
import os
import pstats
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2411_09287_b200.runtime import Session  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 16
N = 1 << L
prog = bench.make_relu_program(N, 16)
xh = torch.from_numpy(np.zeros(N, dtype=np.int64)).pin_memory()
for i in range(2):
    Session(seed=i).run(prog, xh, True)
torch.cuda.synchronize()
profs = {}


def wrapped(party, *a):
    if party.role != 1:          # one profiler at a time (3.12): party 1's thread
        return prog(party, *a)
    pr = cProfile.Profile()
    pr.enable()
    try:
        return prog(party, *a)
    finally:
        pr.disable()
        profs[party.role] = pr


Session(seed=9).run(wrapped, xh, True)
st = pstats.Stats(profs[1])
out = io.StringIO()
st.stream = out
st.sort_stats("tottime").print_stats(30)
print(out.getvalue()[:6000])
