"""Per-party-thread cProfile of the secure-ReLU program (diagnostic)."""
import cProfile, pstats, sys, os, time, io
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, bench
from paper_2411_09287_b200.runtime import Session
N = 1 << int(sys.argv[1]); d = 16
check = len(sys.argv) > 2 and sys.argv[2] == "check"
rng = np.random.default_rng(1)
xv = np.trunc(rng.normal(0, 4, N) * 2 ** 16).astype(np.int64)
xh = torch.from_numpy(xv).pin_memory()
prog = bench.make_relu_program(N, d)
profs = []
def wrapped(party, *a):
    pr = cProfile.Profile()
    profs.append(pr)
    pr.enable()
    try:
        return prog(party, *a)
    finally:
        pr.disable()
keys = ("num_device_alloc", "num_device_free", "num_alloc_retries", "num_sync_all_streams")
for i in range(6):
    s0 = torch.cuda.memory_stats()
    torch.cuda.synchronize()
    t = time.perf_counter()
    profs.clear()
    Session(seed=10 + i).run(wrapped if i == 5 else prog, xh, check)
    torch.cuda.synchronize()
    s1 = torch.cuda.memory_stats()
    print(i, f"{(time.perf_counter() - t) * 1e3:.1f} ms", {k: s1.get(k, 0) - s0.get(k, 0) for k in keys}, flush=True)
st = pstats.Stats(profs[0])
for p in profs[1:]:
    st.add(p)
st.sort_stats("tottime").print_stats(35)
