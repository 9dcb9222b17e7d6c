"""d = 64 dense-level fold (r3_vfy_level_fold, tensor-core form): timing per
role at level-3 size and bit-equality against the CUDA-core form of the
same entry point (a 16-byte-misaligned view forces the CUDA-core kernel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_09287_b200 import _lib, grvec  # noqa: E402


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def fold(role, V, N, acc):
    xa, xb, ya, yb = V
    _lib.call("r3_vfy_level_fold", role, xa.data_ptr(), xb.data_ptr() if role else None, ya.data_ptr(),
              yb.data_ptr() if role else None, N, 64, acc[0].data_ptr(), acc[1].data_ptr(), _lib.stream())


def rand(rows):
    return torch.randint(-2**62, 2**62, (rows, 64), dtype=torch.int64, device="cuda")


for rows in [int(a) for a in (sys.argv[1:] or ["4194304", "1048576", "70001"])]:
    V = [rand(rows) for _ in range(4)]
    acc = grvec.zeros((2, 127))
    for role in (0, 1, 2):
        ms = timeit(lambda: fold(role, V, rows, acc))
        byts = (2 if role == 0 else 4) * rows * 512
        print(f"rows={rows:8d} role {role}: {ms:7.3f} ms  ({byts / ms / 1e6:7.1f} GB/s of distinct operand bytes)")
    if rows <= (1 << 21):
        # CUDA-core reference: the same folds over 8190-row slices (below the
        # tensor-core threshold) accumulated into one output
        for role in (0, 1, 2):
            a1 = grvec.zeros((2, 127))
            a2 = grvec.zeros((2, 127))
            fold(role, V, rows, a1)
            for r0 in range(0, rows, 8190):
                r1 = min(rows, r0 + 8190)
                fold(role, [v[r0:r1] for v in V], r1 - r0, a2)
            torch.cuda.synchronize()
            assert torch.equal(a1, a2), f"role {role} rows {rows}: tc fold != CUDA-core fold"
        print(f"rows={rows:8d}: tensor-core folds equal the CUDA-core folds (roles 0-2)")
