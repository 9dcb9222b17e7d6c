"""cProfile inside each simulated party's thread (the coop engine runs the
parties on their own threads; one profiler per thread, merged).  Time a
party spends parked on the baton shows up under lock.acquire.

    python tools/party_cprofile.py relu|relu_v|mulv LOG2N [sort] [n]
"""
import cProfile, io, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, bench
from paper_2411_09287_b200.runtime import Session
from paper_2411_09287_b200 import verify

kind, lg = sys.argv[1], int(sys.argv[2])
sort = sys.argv[3] if len(sys.argv) > 3 else "tottime"
nshow = int(sys.argv[4]) if len(sys.argv) > 4 else 60
N = 1 << lg
if kind.startswith("relu"):
    rng = np.random.default_rng(1)
    xh = torch.from_numpy(np.trunc(rng.normal(0, 4, N) * 2 ** 16).astype(np.int64)).pin_memory()
    base = bench.make_relu_program(N, 16)
    args = (xh, kind == "relu_v")
else:
    base, _ = bench.make_programs(N, 64, verify.pick_r(N, 64, 64))
    args = ()
profs = []

def prog(party, *a):
    pr = cProfile.Profile()
    profs.append(pr)
    pr.enable()
    try:
        return base(party, *a)
    finally:
        pr.disable()

for i in range(3):
    Session(seed=i).run(base, *args)
torch.cuda.synchronize()
profs.clear()
import time
t0 = time.perf_counter()
for i in range(3):
    Session(seed=10 + i).run(prog, *args)
torch.cuda.synchronize()
print(f"{(time.perf_counter() - t0) / 3 * 1e3:.1f} ms/session (profiled)")
st = pstats.Stats(profs[0])
for p in profs[1:]:
    st.add(p)
st.sort_stats(sort).print_stats(nshow)
