"""Device memory along the structured dot-log verification of a verified
LeNet-28 batch (allocated / peak GiB after each reduction round, the
materialisation and the tail), per party.  Diagnostic only.

    python tools/dots_mem.py BATCH
"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2411_09287_b200 import ppml, verify  # noqa: E402
from paper_2411_09287_b200.runtime import Session  # noqa: E402

G = 2 ** 30
ev = []
active = {"on": False}


def wrap(name):
    orig = getattr(verify, name)

    def inner(party, *a, **k):
        out = orig(party, *a, **k)
        if active["on"]:
            torch.cuda.synchronize()
            ev.append((party.role, name, torch.cuda.memory_allocated() / G, torch.cuda.max_memory_allocated() / G))
        return out
    setattr(verify, name, inner)


for n in ("_reduction_round", "_verify_tail", "_powers"):
    wrap(n)
orig_dots = verify._verify_dots_structured


def dots(party, *a, **k):
    if party.role == 0:
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        ev.append((0, "start", torch.cuda.memory_allocated() / G, 0.0))
    active["on"] = True
    out = orig_dots(party, *a, **k)
    return out


verify._verify_dots_structured = dots
orig_mat = verify._FCBatch.materialise


def mat(self, gr):
    torch.cuda.synchronize()
    b = torch.cuda.memory_allocated() / G
    out = orig_mat(self, gr)
    torch.cuda.synchronize()
    ev.append((-1, f"FC.materialise M={self.M} K={self.K} N={self.N}", b, torch.cuda.max_memory_allocated() / G))
    return out


verify._FCBatch.materialise = mat


def wrap_m(cls, name):
    orig = getattr(cls, name)

    def inner(self, *a, **k):
        torch.cuda.synchronize()
        b = torch.cuda.memory_allocated() / G
        out = orig(self, *a, **k)
        torch.cuda.synchronize()
        tag = f"M={self.M} K={self.K} N={self.N}" if hasattr(self, "M") else \
            f"len={self.length()} base={self.base is not None}"
        ev.append((-1, f"{cls.__name__[1:]}.{name} {tag}"[:44], b, torch.cuda.memory_allocated() / G))
        return out
    setattr(cls, name, inner)


for cls in (verify._FCBatch, verify._DenseBatch):
    for n in ("folds", "reduce"):
        wrap_m(cls, n)
B = int(sys.argv[1])
model = ppml.lenet28_model(np.random.default_rng(0))
imgs = np.random.default_rng(1).normal(0, 1, (B, int(np.prod(model.input_shape))))
Session(seed=1).run(lambda p: ppml.infer_batch(p, model, imgs, ppml.InferConfig(d=16)))
for role, name, a, pk in ev:
    print(f"P{role:2d} {name:44s} alloc {a:7.2f}  {'after' if role < 0 else 'peak '} {pk:7.2f}")
