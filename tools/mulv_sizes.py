"""Verified-multiplication throughput and peak device memory per batch size
on one GPU (the config-2 sweep 2^20..2^28): one warm-up session, then the
median of a few timed sessions per size; stops at the first size that does
not fit.

    python tools/mulv_sizes.py [--lo 20] [--hi 28] [--d 64]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_09287_b200 import verify  # noqa: E402
from paper_2411_09287_b200.runtime import Session  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lo", type=int, default=20)
    ap.add_argument("--hi", type=int, default=28)
    ap.add_argument("--d", type=int, default=64)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    for lg in range(a.lo, a.hi + 1):
        N = 1 << lg
        R = verify.pick_r(N, 64, a.d)
        prog, _ = bench.make_programs(N, a.d, R)
        torch.cuda.empty_cache()
        torch.cuda.reset_peak_memory_stats()
        try:
            ok = Session(seed=1).run(prog)
            times = []
            for i in range(a.reps):
                torch.cuda.synchronize()
                t = time.perf_counter()
                ok = Session(seed=2 + i).run(prog)
                torch.cuda.synchronize()
                times.append(time.perf_counter() - t)
        except torch.OutOfMemoryError as e:
            print(json.dumps({"log2n": lg, "oom": str(e).splitlines()[0][:160]}), flush=True)
            break
        times.sort()
        dt = times[len(times) // 2]
        print(json.dumps({"log2n": lg, "R": R, "verdicts": [bool(v) for v in ok], "ms": round(dt * 1e3, 2),
                          "mults_per_s": N / dt,
                          "peak_gib": round(torch.cuda.max_memory_allocated() / 2 ** 30, 2)}), flush=True)


if __name__ == "__main__":
    main()
