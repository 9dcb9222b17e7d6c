"""Census of the elementwise launches of one mulv step: (op, n words) ->
launches, summed device time (CUDA events per call), with the Python call
site that issued them.  Diagnostic only.

    python tools/ew_census.py [log2n]
"""
import collections, os, sys, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
from paper_2411_09287_b200 import _lib, verify
from paper_2411_09287_b200.runtime import Session

L = int(sys.argv[1]) if len(sys.argv) > 1 else 24
N = 1 << L
prog, _ = bench.make_programs(N, 64, verify.pick_r(N, 64, 64))
for i in range(2):
    Session(seed=i).run(prog)
torch.cuda.synchronize()
ev = []

def hook(name, args, run):
    if not name.startswith("r3_ew"):
        return run()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); rc = run(); b.record()
    if name == "r3_ew_flat":
        key = (name, int(args[0]), int(args[1]))
    elif name == "r3_ew_multi":
        key = (name, int(args[0]), int(args[1]) * int(args[2]))
    else:
        key = (name, int(args[0]), 0)
    st = [f for f in traceback.extract_stack(limit=12) if "paper_2411_09287_b200" in f.filename
          and "_lib.py" not in f.filename and "grvec.py" not in f.filename]
    site = f"{os.path.basename(st[-1].filename)}:{st[-1].lineno}:{st[-1].name}" if st else "?"
    ev.append((key, site, a, b))
    return rc

_lib.CALL_HOOK = hook
Session(seed=99).run(prog)
torch.cuda.synchronize()
_lib.CALL_HOOK = None
agg = collections.defaultdict(lambda: [0, 0.0])
for key, site, a, b in ev:
    k = (key[0], key[1], key[2] if key[2] >= 4096 else "<4096", site)
    agg[k][0] += 1
    agg[k][1] += a.elapsed_time(b)
for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:40]:
    print(f"{ms:8.3f} ms  x{n:4d}  {k}")
print("total", sum(v[1] for v in agg.values()), "ms", sum(v[0] for v in agg.values()), "launches")
