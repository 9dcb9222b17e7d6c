"""Verification cost model restated (reference verify.py:49-87) -- test
infrastructure only (the CPU baseline picks R the way the reference does)."""

import math

PROFILES = {"lan": (0.2, 1e9), "man": (12.0, 1e8), "wan": (80.0, 4e7)}


def online_bits(g, R, ell, d):
    return (5 * R + 3 + math.ceil(g / 2 ** R)) * ell * d


def offline_bits(g, R, ell, d):
    return (R + math.ceil(g / 2 ** R)) * ell * d


def pick_r(g, ell, d, profile="lan", r_max=24):
    if g <= 1:
        return 0
    rtt, bw = PROFILES[profile]
    costs = [((R + 2) * rtt + (online_bits(g, R, ell, d) + offline_bits(g, R, ell, d)) / bw * 1e3, R)
             for R in range(min(r_max, int(math.log2(g))) + 1)]
    return min(costs)[1]
