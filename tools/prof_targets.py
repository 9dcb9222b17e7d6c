"""Launch each hot kernel at its bench shape once (for ncu --set full)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
from paper_2411_09287_b200 import verify, grvec
from paper_2411_09287_b200.runtime import Session
N = 1 << 22
mulv, _ = bench.make_programs(N, 64, verify.pick_r(N, 64, 64))
Session(seed=1).run(mulv)            # level_fold / matmul2_tc / l1_fold / l2_fold / prf
n = 4096
X = torch.randint(-2**62, 2**62, (n, n), dtype=torch.int64, device="cuda")
ta = grvec.limb_tiles_a(X); tb = grvec.limb_tiles_b(X)
grvec.u64_gemm([(ta, tb, n)], n, n)   # share-matmul GEMM
bench.matmul_c3(2048, 1)             # prf_bits_packed at 2^22 lanes
torch.cuda.synchronize()
