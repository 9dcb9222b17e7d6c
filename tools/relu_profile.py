"""cProfile of the secure-ReLU program (diagnostic; in 3.12 the profiler
sees the party threads too)."""
import cProfile, pstats, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, bench
from paper_2411_09287_b200.runtime import Session
N = 1 << int(sys.argv[1]); d = 16
check = len(sys.argv) > 2 and sys.argv[2] == "check"
sort = sys.argv[3] if len(sys.argv) > 3 else "tottime"
rng = np.random.default_rng(1)
xv = np.trunc(rng.normal(0, 4, N) * 2 ** 16).astype(np.int64)
xh = torch.from_numpy(xv).pin_memory()
prog = bench.make_relu_program(N, d)
for i in range(3):
    Session(seed=10 + i).run(prog, xh, check)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
Session(seed=5).run(prog, xh, check)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats(sort).print_stats(45)
