"""Per-entry-point GPU time of one batched private-inference session.
    python tools/ppml_breakdown.py mlp|lenet BATCH [check]"""
import collections
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2411_09287_b200 import _lib, ppml  # noqa: E402
from paper_2411_09287_b200.runtime import Session  # noqa: E402

name, B = sys.argv[1], int(sys.argv[2])
check = len(sys.argv) > 3
model = (ppml.secureml_model if name == "mlp" else ppml.lenet28_model)(np.random.default_rng(0))
imgs = np.random.default_rng(0).normal(0, 1, (B, int(np.prod(model.input_shape))))
cfg = ppml.InferConfig(check=check)
prog = lambda party: ppml.infer_batch(party, model, imgs, cfg)
Session(seed=1).run(prog)
torch.cuda.synchronize()
ev = []


SITE = os.environ.get("SITE_OF")   # entry point whose call sites to list


def hook(nm, args, run):
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    rc = run()
    e.record()
    where = ""
    if nm == SITE:
        import traceback
        fr = [f for f in traceback.extract_stack()[:-2] if "paper_2411_09287_b200" in f.filename]
        where = " <- ".join(f"{os.path.basename(f.filename)}:{f.lineno}:{f.name}" for f in fr[-3:][::-1])
    ev.append((nm, s, e, where))
    return rc


_lib.CALL_HOOK = hook
t0 = time.perf_counter()
Session(seed=2).run(prog)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
_lib.CALL_HOOK = None
tot, cnt = collections.Counter(), collections.Counter()
sites = collections.Counter()
for nm, s, e, w in ev:
    tot[nm] += s.elapsed_time(e)
    cnt[nm] += 1
    if w:
        sites[w] += s.elapsed_time(e)
print(f"{name} B={B} check={check}: wall {wall * 1e3:.1f} ms, library GPU {sum(tot.values()):.1f} ms in {len(ev)} calls,"
      f" peak mem {torch.cuda.max_memory_allocated() / 2**30:.1f} GiB")
for k, v in tot.most_common(14):
    print(f"  {k:26s} {v:9.2f} ms  calls={cnt[k]}")
if SITE:
    print(f"{SITE} by call site:")
    for w, v in sites.most_common(12):
        print(f"  {v:8.2f} ms  {w}")
