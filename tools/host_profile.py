"""cProfile of the host side of one mulv session (diagnostic)."""
import cProfile, pstats, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
from paper_2411_09287_b200 import verify
from paper_2411_09287_b200.runtime import Session
L = int(sys.argv[1]); d = int(sys.argv[2]); eng = sys.argv[3] if len(sys.argv) > 3 else "coop"
N = 1 << L
mulv, _ = bench.make_programs(N, d, verify.pick_r(N, 64, d))
for i in range(2):
    Session(seed=i, engine=eng).run(mulv)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
Session(seed=5, engine=eng).run(mulv)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
st.sort_stats("cumulative").print_stats(60)
