"""cProfile of ONE simulated party's thread (P1: it carries the most work)
over several sessions of a small verified program -- the host-bound regime
where every verification level costs protocol-driver time.  Diagnostic only.

    python tools/party_cprofile.py mulv 20 [tottime|cumtime] [role|all]
"""

import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_09287_b200 import verify  # noqa: E402
from paper_2411_09287_b200.runtime import Session  # noqa: E402


def main():
    kind, lg = sys.argv[1], int(sys.argv[2])
    sort = sys.argv[3] if len(sys.argv) > 3 else "tottime"
    role = sys.argv[4] if len(sys.argv) > 4 else "1"      # a party index or "all"
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
    prs = {r: cProfile.Profile() for r in range(3)}
    roles = range(3) if role == "all" else [int(role)]

    def wrapped(party, *a):
        if party.role not in roles:
            return prog(party, *a)
        pr = prs[party.role]
        pr.enable()
        try:
            return prog(party, *a)
        finally:
            pr.disable()

    if role == "all":
        # Python 3.12's profiler hooks every thread (sys.monitoring): one
        # profiler around the sessions covers all three party threads
        pr = prs[0]
        pr.enable()
        for i in range(5):
            Session(seed=10 + i).run(prog, *args)
        torch.cuda.synchronize()
        pr.disable()
        st = pstats.Stats(pr)
    else:
        for i in range(5):
            Session(seed=10 + i).run(wrapped, *args)
        torch.cuda.synchronize()
        st = pstats.Stats(prs[roles[0]])
    st.sort_stats(sort).print_stats(60)


if __name__ == "__main__":
    main()
