"""Four r^(4j) tables: one r3_gr_matmul_q_tc pass vs four rows_times calls."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2411_09287_b200 import grvec  # noqa: E402
from paper_2411_09287_b200.rings import modulus_for_degree  # noqa: E402

rows = 1 << 22
mod = modulus_for_degree(64)
P = torch.randint(-2**62, 2**62, (rows, 64), dtype=torch.int64, device="cuda")
Ms = [grvec.gr_mulmat(torch.randint(-2**62, 2**62, (1, 64), dtype=torch.int64, device="cuda"), mod) for _ in range(4)]
outs = [torch.empty((rows, 64), dtype=torch.int64, device="cuda") for _ in range(4)]


def t(name, fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{name:22s} {ms:.3f} ms  {rows * 512 * 5 / ms / 1e6:.0f} GB/s algorithmic (1 read + 4 writes)")


t("matmul_q (1 pass)", lambda: grvec.rows_times_multi(P, Ms, rows, 64, outs))
t("4 x rows_times", lambda: [grvec.rows_times(P, M, rows, 64, out=o) for M, o in zip(Ms, outs)])
