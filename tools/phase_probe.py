"""Wall-clock split of one small mulv session (host fixed costs): session
construction, PRE, ONLINE, verification, teardown.

    python tools/phase_probe.py [log2n]
"""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2411_09287_b200 import gates, verify  # noqa: E402
from paper_2411_09287_b200.runtime import Session  # noqa: E402
from paper_2411_09287_b200.sharing import Ring, shc_random  # noqa: E402
from paper_2411_09287_b200.transport import Phase  # noqa: E402

N = 1 << int(sys.argv[1] if len(sys.argv) > 1 else 16)
d = 64
R = verify.pick_r(N, 64, d)
marks = {}


def mark(party, name):
    if party.role == 0:
        torch.cuda.synchronize()
        marks[name] = time.perf_counter()


def prog(party):
    mark(party, "start")
    ring = Ring(64)
    party.enter_phase(Phase.PRE)
    x = shc_random(party, N, ring)
    y = shc_random(party, N, ring)
    g = gates.mul_prepare(party, x.mask, y.mask, N)
    mark(party, "pre_gates")
    verify.prepare_verification(party, d=d, r_max=max(R, 1))
    mark(party, "prep_vfy")
    party.round_barrier()
    party.enter_phase(Phase.ONLINE)
    gates.mul_finish(party, g, x, y)
    party.round_barrier()
    mark(party, "online")
    party.enter_phase(Phase.POST)
    ok = verify.batch_verify_muls(party, 64, d=d, R=R)
    mark(party, "verify")
    return ok


for rep in range(4):
    t0 = time.perf_counter()
    s = Session(seed=rep)
    t1 = time.perf_counter()
    s.run(prog)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    del s
    t3 = time.perf_counter()
    m = marks
    print(f"N=2^{N.bit_length()-1} R={R}: ctor {1e3*(t1-t0):.2f}  to-start {1e3*(m['start']-t1):.2f}  "
          f"pre-gates {1e3*(m['pre_gates']-m['start']):.2f}  prep-vfy {1e3*(m['prep_vfy']-m['pre_gates']):.2f}  "
          f"online {1e3*(m['online']-m['prep_vfy']):.2f}  verify {1e3*(m['verify']-m['online']):.2f}  "
          f"end {1e3*(t2-m['verify']):.2f}  del {1e3*(t3-t2):.2f}  total {1e3*(t3-t0):.2f} ms")
