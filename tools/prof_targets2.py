"""Launch the d = 64 verification kernels (line evaluations, level fold) at
level-3 size of an N = 2^24 session and one 4096^3 u64 GEMM, for
ncu --set full (-s 2 skips the warm-up launches of the first two).  The
line evaluation is the multi-job form the protocol issues: one party's x
and y components of a level in one launch (r3_gr_matmul2_tc_multi)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2411_09287_b200 import _lib, grvec  # noqa: E402
from paper_2411_09287_b200.rings import modulus_for_degree  # noqa: E402

rows = 1 << 22
mod = modulus_for_degree(64)
X = torch.randint(-2**62, 2**62, (rows, 64), dtype=torch.int64, device="cuda")
Y = torch.randint(-2**62, 2**62, (rows, 64), dtype=torch.int64, device="cuda")
z = torch.randint(-2**62, 2**62, (1, 64), dtype=torch.int64, device="cuda")
Ma = grvec.gr_mulmat(z, mod)
Mb = grvec.gr_mulmat(z + 1, mod)
n0 = rows // 2
acc1 = torch.zeros(127, dtype=torch.int64, device="cuda")
acc2 = torch.zeros(127, dtype=torch.int64, device="cuda")
def line_evals():
    # x and y of one party: out = f0 . Ma + f1 . Mb over the even / odd rows
    grvec.rows_times2_batch([(X[0::2], X[1::2], n0, n0), (Y[0::2], Y[1::2], n0, n0)], Ma, Mb, 64)


def fold():
    _lib.call("r3_vfy_level_fold", 1, X.data_ptr(), Y.data_ptr(), Y.data_ptr(), X.data_ptr(), rows, 64,
              acc1.data_ptr(), acc2.data_ptr(), _lib.stream())


for _ in range(2):   # warm-up (skipped by ncu -s 2 ... order: mm2, lf, mm2, lf)
    line_evals()
    fold()
line_evals()
fold()
torch.cuda.synchronize()
del X, Y
n = 4096
A = torch.randint(-2**62, 2**62, (n, n), dtype=torch.int64, device="cuda")
ta = grvec.limb_tiles_a(A)
tb = grvec.limb_tiles_b(A)
grvec.u64_gemm([(ta, tb, n)], n, n)
torch.cuda.synchronize()
