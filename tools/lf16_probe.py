"""One d = 16 CUDA-core level fold at the level-3 size of a 2^20-lane ReLU's
arithmetic multiplication log (for ncu and timing)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2411_09287_b200 import _lib  # noqa: E402

d = 16
rows = 67 * (1 << 20) // 4
X = torch.randint(-2**62, 2**62, (rows, d), dtype=torch.int64, device="cuda")
Y = torch.randint(-2**62, 2**62, (rows, d), dtype=torch.int64, device="cuda")
acc1 = torch.zeros(2 * d - 1, dtype=torch.int64, device="cuda")
acc2 = torch.zeros(2 * d - 1, dtype=torch.int64, device="cuda")
for role in (0, 1, 2):
    _lib.call("r3_vfy_level_fold", role, X.data_ptr(), Y.data_ptr(), Y.data_ptr(), X.data_ptr(), rows, d,
              acc1.data_ptr(), acc2.data_ptr(), _lib.stream())
torch.cuda.synchronize()
for role in (0, 1, 2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.call("r3_vfy_level_fold", role, X.data_ptr(), Y.data_ptr(), Y.data_ptr(), X.data_ptr(), rows, d,
              acc1.data_ptr(), acc2.data_ptr(), _lib.stream())
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    nb = (2 if role == 0 else 4) * rows * d * 8
    print(f"level_fold d=16 role {role} rows {rows}: {ms:.3f} ms, {nb / ms / 1e6:.0f} GB/s")
