"""Peak device memory of verified workloads and what the gate logs hold at
the end of the online phase (bytes per log kind), to see what bounds the
verified batch.

    python tools/mem_probe.py relu 65536
    python tools/mem_probe.py lenet 16
"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_09287_b200 import ppml, verify  # noqa: E402
from paper_2411_09287_b200.runtime import Session  # noqa: E402


def log_bytes(party):
    out = {}
    for key, logs in party.logs.items():
        for kind in ("muls", "dots"):
            out[f"{key}.{kind}"] = sum(_tb(rec) for rec in getattr(logs, kind))
            out[f"{key}.{kind}.lanes"] = sum(getattr(rec, "lanes", 0) for rec in getattr(logs, kind))
    return out


def _tb(v, seen=None):
    if isinstance(v, torch.Tensor):
        return v.numel() * v.element_size()
    if hasattr(v, "__dict__"):
        return sum(_tb(x) for x in vars(v).values())
    if isinstance(v, (list, tuple)):
        return sum(_tb(x) for x in v)
    return 0


def main():
    what, n = sys.argv[1], int(sys.argv[2])
    snap = {}
    orig = verify.verify_session

    def spy(party, *a, **k):
        if party.role == 0:
            torch.cuda.synchronize()
            snap["alloc_at_post_gib"] = torch.cuda.memory_allocated() / 2 ** 30
            snap["logs_gib"] = {r: {k2: (v / 2 ** 30 if not k2.endswith("lanes") else v)
                                     for k2, v in log_bytes(p).items()} for r, p in enumerate(party.sess.parties)}
        return orig(party, *a, **k)

    verify.verify_session = spy
    if what == "relu":
        xv = np.trunc(np.random.default_rng(1).normal(0, 4, n) * 2 ** 16).astype(np.int64)
        prog = bench.make_relu_program(n, 16)
        torch.cuda.reset_peak_memory_stats()
        Session(seed=1).run(prog, torch.from_numpy(xv), True)
    else:
        model = ppml.lenet28_model(np.random.default_rng(0)) if what == "lenet" else ppml.secureml_model(np.random.default_rng(0))
        imgs = np.random.default_rng(1).normal(0, 1, (n, int(np.prod(model.input_shape))))
        torch.cuda.reset_peak_memory_stats()
        Session(seed=1).run(lambda p: ppml.infer_batch(p, model, imgs, ppml.InferConfig(d=16)))
    snap["peak_gib"] = torch.cuda.max_memory_allocated() / 2 ** 30
    print(what, n, snap)


if __name__ == "__main__":
    main()
