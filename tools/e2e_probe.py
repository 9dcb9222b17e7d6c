"""Wall time split of the bench's e2e step (diagnostic)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2411_09287_b200 import verify  # noqa: E402
from paper_2411_09287_b200.runtime import Session  # noqa: E402

N = 1 << 24
R = verify.pick_r(N, 64, 64)
mulv, e2e = bench.make_programs(N, 64, R)
g = np.random.default_rng(0)
xh = torch.from_numpy(g.integers(0, 2**63, N, dtype=np.int64)).pin_memory()
yh = torch.from_numpy(g.integers(0, 2**63, N, dtype=np.int64)).pin_memory()
pin = torch.empty(N, dtype=torch.int64, pin_memory=True)
for _ in range(2):
    Session(seed=1).run(e2e, xh, yh)
    Session(seed=1).run(mulv)
torch.cuda.synchronize()
for name, fn in (("mulv", lambda: Session(seed=3).run(mulv)),
                 ("e2e-session", lambda: Session(seed=3).run(e2e, xh, yh)),
                 ("e2e+d2h", lambda: Session(seed=3).run(e2e, xh, yh)[0].cpu()),
                 ("e2e+pinned", lambda: pin.copy_(Session(seed=3).run(e2e, xh, yh)[0], non_blocking=True))):
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"{name:12s} {min(ts) * 1e3:8.1f} ms")
t0 = time.perf_counter()
a = xh.to("cuda", non_blocking=False)
torch.cuda.synchronize()
print(f"h2d 128MB {1e3 * (time.perf_counter() - t0):.1f} ms")
t0 = time.perf_counter()
b = a.cpu()
print(f"d2h 128MB {1e3 * (time.perf_counter() - t0):.1f} ms")
