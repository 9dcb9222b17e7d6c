"""Acceptance criterion 4 of the reference (tests/test_acceptance.py:160-208)
on the GPU backend: 4 x 1000 injected-error trials of Pi_mulv (d = 16,
R = 2, 64 gates) plus 1000 d = 1 ring-attack control trials, each trial one
full three-party session.  Worker processes share the GPU (each its own
CUDA context); prints one JSON line with misses, the control acceptance rate
and wall-clock seconds (the reference's bar: <= 30 misses per mode, control
0.50 +/- 0.05, under 300 s).

    python tools/soundness_mc.py [--trials 1000] [--workers 4]
"""

import argparse
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def _chunk(args):
    mode, lo, hi = args
    from paper_2411_09287_b200.cli import run_soundness_trial
    from test_gpu_circuit import _trial_args
    bad = 0
    for t in range(lo, hi):
        if mode == "control":
            bad += not run_soundness_trial((5 << 20) + t, 64, 1, 0, 64, 1 << 63, "gamma", 0)
        else:
            seed, delta, site, lane = _trial_args(mode, t)
            bad += not run_soundness_trial(seed, 64, 16, 2, 64, delta, site, lane)
    return mode, bad


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=1000)
    ap.add_argument("--workers", type=int, default=4)
    a = ap.parse_args()
    step = max(1, a.trials // (4 * a.workers))
    jobs = [(m, lo, min(lo + step, a.trials)) for m in ("random", "msb", "gamma", "mz", "control")
            for lo in range(0, a.trials, step)]
    t0 = time.perf_counter()
    res = {m: 0 for m in ("random", "msb", "gamma", "mz", "control")}
    with mp.get_context("spawn").Pool(a.workers) as pool:
        for mode, bad in pool.imap_unordered(_chunk, jobs):
            res[mode] += bad
    dt = time.perf_counter() - t0
    control = res.pop("control") / a.trials
    ok = all(v <= 0.03 * a.trials for v in res.values()) and 0.45 <= control <= 0.55
    print(json.dumps({"criterion": 4, "trials_per_mode": a.trials, "workers": a.workers,
                      "misses": res, "control_acceptance": control, "seconds": round(dt, 1),
                      "sessions": 5 * a.trials, "sessions_per_s": round(5 * a.trials / dt, 1),
                      "pass": ok and dt < 300}))


if __name__ == "__main__":
    main()
