"""Micro-costs of the host path (diagnostic): allocation, ctypes launch,
baton switches per session."""
import sys, os, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, bench
from paper_2411_09287_b200 import _lib, grvec, runtime
from paper_2411_09287_b200.runtime import Session
dev = torch.device("cuda", 0)
torch.empty(1, device=dev)
def bench_empty(tag):
    n = 20000
    t = time.perf_counter()
    for _ in range(n):
        torch.empty(65536, dtype=torch.int64, device=dev)
    print(tag, "torch.empty", (time.perf_counter() - t) / n * 1e6, "us", flush=True)
    a = torch.zeros(65536, dtype=torch.int64, device=dev)
    t = time.perf_counter()
    for _ in range(n):
        grvec.ew(grvec.XOR, a, a, 1)
    torch.cuda.synchronize()
    print(tag, "grvec.ew", (time.perf_counter() - t) / n * 1e6, "us", flush=True)
    o = torch.empty_like(a)
    t = time.perf_counter()
    for _ in range(n):
        torch.bitwise_xor(a, a, out=o)
    torch.cuda.synchronize()
    print(tag, "torch xor out=", (time.perf_counter() - t) / n * 1e6, "us", flush=True)
bench_empty("main")
th = threading.Thread(target=lambda: (torch.cuda.set_device(0), bench_empty("thread")))
th.start(); th.join()
# count baton resumes in one relu session
cnt = [0]
orig = runtime._Baton.resume
def resume(self, i):
    cnt[0] += 1
    return orig(self, i)
runtime._Baton.resume = resume
N = 1 << 16
xv = np.zeros(N, dtype=np.int64)
xh = torch.from_numpy(xv).pin_memory()
prog = bench.make_relu_program(N, 16)
for check in (False, True):
    cnt[0] = 0
    Session(seed=3).run(prog, xh, check)
    print("relu check" if check else "relu exec", "resumes", cnt[0], flush=True)
mulv, _ = bench.make_programs(1 << 20, 64, 15)
cnt[0] = 0
Session(seed=3).run(mulv)
print("mulv 2^20 resumes", cnt[0])
