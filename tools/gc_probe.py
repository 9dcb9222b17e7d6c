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
