"""Launch the d = 64 tensor-core verification kernels once at level-3 size of
an N = 2^24 session (for ncu --set full)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2411_09287_b200 import _lib, grvec  # noqa: E402
from paper_2411_09287_b200.rings import modulus_for_degree  # noqa: E402

rows = 1 << 22   # level-3 vectors of N = 2^24 (N / 4 rows)
mod = modulus_for_degree(64)
X = torch.randint(-2**62, 2**62, (rows, 64), dtype=torch.int64, device="cuda")
Y = torch.randint(-2**62, 2**62, (rows, 64), dtype=torch.int64, device="cuda")
z = torch.randint(-2**62, 2**62, (1, 64), dtype=torch.int64, device="cuda")
Ma = grvec.gr_mulmat(z, mod)
Mb = grvec.gr_mulmat(z + 1, mod)
ev, od = X[0::2], X[1::2]
n0 = rows // 2
out = grvec.empty((n0, 64))
for _ in range(2):
    _lib.call("r3_gr_matmul2_tc", ev.data_ptr(), 128, n0, od.data_ptr(), 128, n0, Ma.data_ptr(),
              Mb.data_ptr(), out.data_ptr(), n0, (1 << 64) - 1, _lib.stream())
acc1 = torch.zeros(127, dtype=torch.int64, device="cuda")
acc2 = torch.zeros(127, dtype=torch.int64, device="cuda")
for role in (1,):
    _lib.call("r3_vfy_level_fold", role, X.data_ptr(), Y.data_ptr(), Y.data_ptr(), X.data_ptr(), rows, 64,
              acc1.data_ptr(), acc2.data_ptr(), _lib.stream())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
_lib.call("r3_gr_matmul2_tc", ev.data_ptr(), 128, n0, od.data_ptr(), 128, n0, Ma.data_ptr(),
          Mb.data_ptr(), out.data_ptr(), n0, (1 << 64) - 1, _lib.stream())
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"matmul2_tc rows {n0}: {ms:.3f} ms, {n0 * 1536 / ms / 1e6:.0f} GB/s algorithmic")
e0.record()
_lib.call("r3_vfy_level_fold", 1, X.data_ptr(), Y.data_ptr(), Y.data_ptr(), X.data_ptr(), rows, 64,
          acc1.data_ptr(), acc2.data_ptr(), _lib.stream())
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"level_fold role1 rows {rows}: {ms:.3f} ms, {rows * 4 * 512 / ms / 1e6:.0f} GB/s algorithmic")
