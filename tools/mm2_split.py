"""Split r3_gr_matmul2_tc time of one mulv step into single-operand calls
(power / line tables) and two-operand calls (level line evaluations)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2411_09287_b200 import _lib, verify  # noqa: E402
from paper_2411_09287_b200.runtime import Session  # noqa: E402

N = 1 << 24
mulv, _ = bench.make_programs(N, 64, verify.pick_r(N, 64, 64))
Session(seed=1).run(mulv)
torch.cuda.synchronize()
ev = []


def hook(name, args, run):
    if name != "r3_gr_matmul2_tc":
        return run()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    rc = run()
    e.record()
    ev.append((args[3] is None, int(args[9]), s, e))
    return rc


_lib.CALL_HOOK = hook
Session(seed=2).run(mulv)
_lib.CALL_HOOK = None
torch.cuda.synchronize()
for single in (True, False):
    sel = [(rows, s.elapsed_time(e)) for sg, rows, s, e in ev if sg == single]
    rows = sum(r for r, _ in sel)
    ms = sum(t for _, t in sel)
    nb = rows * 512 * (2 if single else 3)
    print(f"{'single-op (tables)' if single else 'two-op (line evals)':22s} calls {len(sel):4d} rows {rows:11d} "
          f"{ms:7.2f} ms {nb / ms / 1e6 if ms else 0:7.0f} GB/s")
    big = sorted(sel, reverse=True)[:3]
    print("   largest:", [(r, round(t, 3)) for r, t in big])
    small = [(r, t) for r, t in sel if r < 148 * 128]
    print(f"   launches under one wave: {len(small)} calls, {sum(t for _, t in small):.2f} ms")
