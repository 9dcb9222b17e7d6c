"""Peak device memory of each verification (mul.arith, dot.arith, mul.bool)
of one verified secure-ReLU session, against the logs held at POST.

    python tools/verify_mem.py LOG2N
    python tools/verify_mem.py lenet BATCH
"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_09287_b200 import ppml, verify  # noqa: E402
from paper_2411_09287_b200.runtime import Session  # noqa: E402

lenet = sys.argv[1] == "lenet"
n = int(sys.argv[2]) if lenet else 1 << int(sys.argv[1])
rows = []
state = {}
for name in ("batch_verify_muls", "batch_verify_dots"):
    orig = getattr(verify, name)

    def wrap(party, base_ell, *a, _orig=orig, _name=name, **k):
        if party.role == 0:
            torch.cuda.synchronize()
            state[_name] = torch.cuda.memory_allocated()
            torch.cuda.reset_peak_memory_stats()
        out = _orig(party, base_ell, *a, **k)
        if party.role == 2:
            torch.cuda.synchronize()
            rows.append((_name, base_ell, state[_name] / 2 ** 30, torch.cuda.max_memory_allocated() / 2 ** 30))
        return out
    setattr(verify, name, wrap)
if lenet:
    model = ppml.lenet28_model(np.random.default_rng(0))
    imgs = np.random.default_rng(1).normal(0, 1, (n, int(np.prod(model.input_shape))))
    Session(seed=1).run(lambda p: ppml.infer_batch(p, model, imgs, ppml.InferConfig(d=16)))
else:
    xv = np.trunc(np.random.default_rng(1).normal(0, 4, n) * 2 ** 16).astype(np.int64)
    Session(seed=1).run(bench.make_relu_program(n, 16), torch.from_numpy(xv), True)
for name, ell, before, peak in rows:
    print(f"{name:18s} ell={ell:2d}: allocated before {before:6.2f} GiB, peak {peak:6.2f} GiB "
          f"({(peak - before) * 2 ** 30 / n / 1024:.1f} KiB per {'image' if lenet else 'ReLU lane'} above the logs)")
