"""Which objects of a finished session survive only through reference cycles
(they hold device memory until the next cyclic GC).  Diagnostic."""
import collections, gc, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, bench
from paper_2411_09287_b200.runtime import Session
N = 1 << 12
xh = torch.zeros(N, dtype=torch.int64).pin_memory()
mulv, e2e = bench.make_programs(N, 16, 3)
relu = bench.make_relu_program(N, 16)
progs = {"mulv": (mulv, ()), "relu": (relu, (xh, False)), "relu_check": (relu, (xh, True))}
gc.collect()
for name, (p, a) in progs.items():
    gc.disable()
    s = Session(seed=1)
    s.run(p, *a)
    del s
    gc.set_debug(gc.DEBUG_SAVEALL)
    n = gc.collect()
    c = collections.Counter(type(o).__name__ for o in gc.garbage)
    print(name, "cyclic garbage", n, c.most_common(12), flush=True)
    gc.garbage.clear()
    gc.set_debug(0)
    gc.enable()

# keystream draws made by only one holder (they stay in prg_shared until
# run() returns)
class Rec(dict):
    def clear(self):
        if self:
            print("   leftover draws", len(self), "bytes", sum(t.numel() * 8 for t in self.values()),
                  sorted({(k[1], k[2]) for k in self})[:6], flush=True)
        super().clear()
for name, (p, a) in progs.items():
    s = Session(seed=1)
    s.prg_shared = Rec()
    for party in s.parties:
        pass
    print(name)
    s.run(p, *a)
