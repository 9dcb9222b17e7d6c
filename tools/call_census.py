"""Census of library calls of one small mulv session by protocol stage and
call site (which Python paths issue the most launches)."""
import collections, os, sys, traceback
sys.path.insert(0, "/root/repo")
import torch, bench
from paper_2411_09287_b200 import _lib, verify
from paper_2411_09287_b200.runtime import Session
N = 1 << 16
prog, _ = bench.make_programs(N, 64, verify.pick_r(N, 64, 64))
Session(seed=1).run(prog)
cnt = collections.Counter()
def hook(name, args, run):
    st = traceback.extract_stack()
    fns = [f.name for f in st if "paper_2411_09287_b200" in f.filename]
    top = next((f for f in fns if f in ("reduce_dimension", "check_inner_product", "_compress_reduce_first", "prepare_verification", "mul_prepare", "mul_finish", "shc_random")), "other")
    where = [f"{os.path.basename(f.filename)}:{f.lineno}:{f.name}" for f in st
             if "paper_2411_09287_b200" in f.filename and "_lib.py" not in f.filename][-4:]
    cnt[(top, name, " <- ".join(where))] += 1
    return run()
_lib.CALL_HOOK = hook
Session(seed=2).run(prog)
_lib.CALL_HOOK = None
tot = collections.Counter()
for (top, name, w), c in cnt.items():
    tot[top] += c
print(tot)
for (top, name, w), c in sorted(cnt.items(), key=lambda kv: -kv[1])[:45]:
    print(f"{c:5d} {top:22s} {name:24s} {w}")
