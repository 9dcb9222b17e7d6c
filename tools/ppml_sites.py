"""GPU time of one library entry point by Python call site, in one verified
batched-inference session (events around each call).

    python tools/ppml_sites.py mlp|lenet BATCH r3_gr_mul
"""
import collections
import os
import sys
import traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2411_09287_b200 import _lib, ppml  # noqa: E402
from paper_2411_09287_b200.runtime import Session  # noqa: E402

name, B, target = sys.argv[1], int(sys.argv[2]), sys.argv[3]
model = (ppml.secureml_model if name == "mlp" else ppml.lenet28_model)(np.random.default_rng(0))
imgs = np.random.default_rng(0).normal(0, 1, (B, int(np.prod(model.input_shape))))
cfg = ppml.InferConfig(check=True)
prog = lambda party: ppml.infer_batch(party, model, imgs, cfg)
Session(seed=1).run(prog)
torch.cuda.synchronize()
ev = []


def hook(n, args, run):
    if n != target:
        return run()
    st = traceback.extract_stack()[:-2]
    where = " <- ".join(f"{os.path.basename(f.filename)}:{f.lineno}:{f.name}" for f in st
                        if "paper_2411_09287_b200" in f.filename and "_lib.py" not in f.filename)
    where = " <- ".join(where.split(" <- ")[-4:])
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    rc = run()
    b.record()
    ev.append((where, a, b, [x for x in args if isinstance(x, int)][:4]))
    return rc


_lib.CALL_HOOK = hook
Session(seed=2).run(prog)
_lib.CALL_HOOK = None
torch.cuda.synchronize()
tot, cnt = collections.Counter(), collections.Counter()
for w, a, b, _ in ev:
    tot[w] += a.elapsed_time(b)
    cnt[w] += 1
for w, v in tot.most_common(12):
    print(f"{v:9.2f} ms  n={cnt[w]:5d}  {w}")
