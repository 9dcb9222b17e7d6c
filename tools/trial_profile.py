"""Host profile of one small soundness trial session (64 gates, d = 16,
R = 2) on the GPU backend: wall time per session and the top cProfile
entries, to find per-session fixed costs.

    python tools/trial_profile.py [--n 40]
"""
import argparse
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=40)
    a = ap.parse_args()
    import torch
    from paper_2411_09287_b200.cli import run_soundness_trial
    for i in range(3):
        run_soundness_trial((1 << 20) + i, 64, 16, 2, 64, 12345, "z", 3)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for i in range(a.n):
        run_soundness_trial((1 << 20) + i, 64, 16, 2, 64, 12345, "z", 3)
    torch.cuda.synchronize()
    print(f"per trial {1e3 * (time.perf_counter() - t) / a.n:.2f} ms")
    pr = cProfile.Profile()
    pr.enable()
    for i in range(a.n):
        run_soundness_trial((1 << 20) + i, 64, 16, 2, 64, 12345, "z", 3)
    pr.disable()
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(25)
    st.sort_stats("cumulative").print_stats(40)


if __name__ == "__main__":
    main()
