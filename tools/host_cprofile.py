"""cProfile of the host protocol driver for one small session (the
host-bound regime: secure ReLU 2^16, mulv 2^20).

    python tools/host_cprofile.py relu|relu_v|mulv LOG2N [sort]
"""
import cProfile, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, bench
from paper_2411_09287_b200.runtime import Session
from paper_2411_09287_b200 import verify

kind, lg = sys.argv[1], int(sys.argv[2])
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
pr = cProfile.Profile()
pr.enable()
for i in range(3):
    Session(seed=10 + i).run(prog, *args)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats(sys.argv[3] if len(sys.argv) > 3 else "tottime").print_stats(45)
