"""Library calls of one program grouped by Python call site (diagnostic).
    python tools/call_sites.py relu|relu_check|mulv [log2n]"""
import collections, sys, os, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, bench
from paper_2411_09287_b200 import _lib, verify
from paper_2411_09287_b200.runtime import Session
what = sys.argv[1]
L = int(sys.argv[2]) if len(sys.argv) > 2 else 16
N = 1 << L
if what.startswith("relu"):
    xh = torch.zeros(N, dtype=torch.int64).pin_memory()
    prog, args = bench.make_relu_program(N, 16), (xh, what == "relu_check")
else:
    prog, args = bench.make_programs(N, 64, verify.pick_r(N, 64, 64))[0], ()
Session(seed=1).run(prog, *args)
sites = collections.Counter()
def hook(name, a, run):
    st = traceback.extract_stack(limit=7)[:-2]
    chain = " < ".join(f"{os.path.basename(f.filename)}:{f.name}:{f.lineno}" for f in reversed(st[-4:]))
    sites[(name, chain)] += 1
    return run()
_lib.CALL_HOOK = hook
Session(seed=2).run(prog, *args)
_lib.CALL_HOOK = None
tot = sum(sites.values())
print("total library calls", tot)
for (name, chain), c in sites.most_common(45):
    print(f"{c:6d} {name:22s} {chain}")
