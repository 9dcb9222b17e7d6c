"""u64 share-matmul GEMM on the tensor cores at 4096^3 (CUDA events)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_09287_b200 import grvec

def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps / 1e3

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
X = torch.randint(-2**62, 2**62, (n, n), dtype=torch.int64, device="cuda")
W = torch.randint(-2**62, 2**62, (n, n), dtype=torch.int64, device="cuda")
ta = grvec.limb_tiles_a(X); tb = grvec.limb_tiles_b(W)
t_split_a = timeit(lambda: grvec.limb_tiles_a(X))
t_split_b = timeit(lambda: grvec.limb_tiles_b(W))
t1 = timeit(lambda: grvec.u64_gemm([(ta, tb, n)], n, n))
t2 = timeit(lambda: grvec.u64_gemm([(ta, tb, n), (ta, tb, n)], n, n))
int8_ops = 2 * 36 * n ** 3
print(f"n={n}: split A {t_split_a*1e3:.3f} ms, split B {t_split_b*1e3:.3f} ms")
print(f"  gemm K=n   {t1*1e3:.3f} ms  {int8_ops/t1/1e12:.1f} int8 TOPS  {n**3/t1/1e12:.3f} T u64MAC/s")
print(f"  gemm K=2n  {t2*1e3:.3f} ms  {2*int8_ops/t2/1e12:.1f} int8 TOPS")
