"""Verified LeNet-28 batch per session: time and peak memory per batch size.

    python tools/lenet_batch_probe.py 64 128 192
"""
import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2411_09287_b200 import ppml
from paper_2411_09287_b200.runtime import Session
model = ppml.lenet28_model(np.random.default_rng(0))
for B in [int(x) for x in sys.argv[1:]]:
    imgs = np.random.default_rng(1).normal(0, 1, (B, int(np.prod(model.input_shape))))
    torch.cuda.reset_peak_memory_stats(); torch.cuda.synchronize()
    t = time.perf_counter()
    try:
        res = Session(seed=3).run(lambda p: ppml.infer_batch(p, model, imgs, ppml.InferConfig(check=True)))
        torch.cuda.synchronize()
        print(f"B={B}: ok={all(res[0][1].values())} {time.perf_counter()-t:.2f} s peak {torch.cuda.max_memory_allocated()/2**30:.1f} GiB", flush=True)
    except torch.OutOfMemoryError as e:
        print(f"B={B}: OOM", flush=True)
    torch.cuda.empty_cache()
