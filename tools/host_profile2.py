"""cProfile of the three party threads of one mulv session (diagnostic)."""
import cProfile, pstats, sys, os, io, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
from paper_2411_09287_b200 import verify
from paper_2411_09287_b200.runtime import Session
L = int(sys.argv[1]); d = int(sys.argv[2])
N = 1 << L
mulv, _ = bench.make_programs(N, d, verify.pick_r(N, 64, d))
for i in range(2):
    Session(seed=i).run(mulv)
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
Session(seed=5).run(mulv)
torch.cuda.synchronize()
pr.disable()
print("wall", time.perf_counter() - t0)
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(30)
