"""Per-entry-point GPU time of one C3 (4096^3 share matmul + trunc) session."""
import collections, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2411_09287_b200 import _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
bench.matmul_c3(n, 1)
ev = []
def hook(name, args, run):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); rc = run(); e.record(); ev.append((name, s, e)); return rc
_lib.CALL_HOOK = hook
r = bench.matmul_c3(n, 1)
_lib.CALL_HOOK = None
torch.cuda.synchronize()
tot = collections.Counter(); cnt = collections.Counter()
for name, s, e in ev:
    tot[name] += s.elapsed_time(e); cnt[name] += 1
print(r["ms_per_matmul"], "ms per matmul (timed step); hooked run GPU time by entry point:")
for k, v in tot.most_common(12):
    print(f"  {k:24s} {v:9.2f} ms calls={cnt[k]}")
