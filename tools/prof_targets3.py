"""One launch each of the round's new tensor-core kernels at bench shapes
(for ncu --set full): the all-party base fold over the r^(4j) table of an
N = 2^24 session (via one mulv session) and a 4096^3 u64 GEMM."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2411_09287_b200 import grvec, verify  # noqa: E402
from paper_2411_09287_b200.runtime import Session  # noqa: E402

N = 1 << 24
mulv, _ = bench.make_programs(N, 64, verify.pick_r(N, 64, 64))
Session(seed=1).run(mulv)
n = 4096
A = torch.randint(-2**62, 2**62, (n, n), dtype=torch.int64, device="cuda")
ta, tb = grvec.limb_tiles_a(A), grvec.limb_tiles_b(A)
grvec.u64_gemm([(ta, tb, n)], n, n)
torch.cuda.synchronize()
