"""Throughput of the d = 16 tensor-core line evaluation and the d = 16
CUDA-core level fold at the level-3 size of a 2^20-lane ReLU log."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2411_09287_b200 import _lib, grvec  # noqa: E402
from paper_2411_09287_b200.rings import modulus_for_degree  # noqa: E402

d = 16
rows = 1 << 24
mod = modulus_for_degree(d)
X = torch.randint(-2**62, 2**62, (rows, d), dtype=torch.int64, device="cuda")
Y = torch.randint(-2**62, 2**62, (rows, d), dtype=torch.int64, device="cuda")
z = torch.randint(-2**62, 2**62, (1, d), dtype=torch.int64, device="cuda")
Ma, Mb = grvec.gr_mulmat(z, mod), grvec.gr_mulmat(z + 1, mod)
n0 = rows // 2
out = grvec.empty((n0, d))
acc1 = torch.zeros(2 * d - 1, dtype=torch.int64, device="cuda")
acc2 = torch.zeros(2 * d - 1, dtype=torch.int64, device="cuda")


def t(fn, nbytes, name):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{name:34s} {ms:7.3f} ms  {nbytes / ms / 1e6:6.0f} GB/s")


t(lambda: _lib.call("r3_gr_matmul2_tc16", X.data_ptr(), 2 * d, n0, X[1:].data_ptr(), 2 * d, n0, Ma.data_ptr(),
                    Mb.data_ptr(), out.data_ptr(), n0, (1 << 64) - 1, _lib.stream()),
  n0 * 3 * 8 * d, "tc16 line eval (2^23 out rows)")
for role in (0, 1):
    t(lambda: _lib.call("r3_vfy_level_fold", role, X.data_ptr(), Y.data_ptr(), Y.data_ptr(), X.data_ptr(), rows,
                        d, acc1.data_ptr(), acc2.data_ptr(), _lib.stream()),
      rows * 8 * d * (2 if role == 0 else 4), f"level_fold d16 role {role} (2^24 rows)")
