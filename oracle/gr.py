"""GR(2^ell, d) arithmetic restated in numpy -- test infrastructure only.

Follows the reference's ring definition (rings.py:180-241, grvec.py:78-167)
with an independent formulation: schoolbook product followed by the sparse
reduction x^d = -g(x) applied top-down (the reference multiplies the high
half by a dense (d-1, d) reduction matrix).  Elements are (n, d) uint64
arrays, constant coefficient first; numpy uint64 arithmetic wraps mod 2^64
and results are masked to ell bits.
"""

from __future__ import annotations

import numpy as np

U = np.uint64

MODULUS_BITS = {  # rings.py:180-188
    1: 0b11, 2: 0b111, 4: 0b10011, 8: 0x11B,
    16: (1 << 16) | (1 << 5) | (1 << 3) | (1 << 1) | 1,
    32: (1 << 32) | (1 << 7) | (1 << 3) | (1 << 2) | 1,
    64: (1 << 64) | (1 << 4) | (1 << 3) | (1 << 1) | 1,
}


def mask_of(ell: int) -> np.uint64:
    return U((1 << ell) - 1)


def low_terms(d: int) -> list[int]:
    return [j for j in range(d) if (MODULUS_BITS[d] >> j) & 1]


def mul(a: np.ndarray, b: np.ndarray, ell: int, d: int) -> np.ndarray:
    """Rowwise product mod f and 2^ell; rows broadcast on axis 0."""
    a = np.asarray(a, dtype=U).reshape(-1, d)
    b = np.asarray(b, dtype=U).reshape(-1, d)
    n = max(a.shape[0], b.shape[0])
    p = np.zeros((n, 2 * d - 1), dtype=U)
    with np.errstate(over="ignore"):
        for i in range(d):
            p[:, i:i + d] += a[:, i:i + 1] * b
        lows = low_terms(d)
        for k in range(2 * d - 2, d - 1, -1):
            top = p[:, k].copy()
            for j in lows:
                p[:, k - d + j] -= top
    return p[:, :d] & mask_of(ell)


def dot(a: np.ndarray, b: np.ndarray, ell: int, d: int) -> np.ndarray:
    """sum_i a_i * b_i as (1, d)."""
    with np.errstate(over="ignore"):
        return (mul(a, b, ell, d).sum(axis=0, dtype=U) & mask_of(ell)).reshape(1, d)


def embed(base: np.ndarray, d: int) -> np.ndarray:
    out = np.zeros((base.shape[0], d), dtype=U)
    out[:, 0] = base
    return out


def const(v: int, ell: int, d: int) -> np.ndarray:
    out = np.zeros((1, d), dtype=U)
    out[0, 0] = U(v & ((1 << ell) - 1))
    return out


def powers(r: np.ndarray, n: int, ell: int, d: int) -> np.ndarray:
    """r^0 .. r^(n-1): powers of r^64 times the first 64 powers."""
    r = np.asarray(r, dtype=U).reshape(1, d)
    T = min(64, max(n, 1))
    small = np.zeros((T, d), dtype=U)
    small[0, 0] = 1
    for i in range(1, T):
        small[i] = mul(small[i - 1:i], r, ell, d)[0]
    if n <= T:
        return small[:n] & mask_of(ell)
    step = mul(small[T - 1:T], r, ell, d)           # r^T
    blocks = (n + T - 1) // T
    out = np.zeros((blocks * T, d), dtype=U)
    big = small[:1].copy()
    for bidx in range(blocks):
        out[bidx * T:(bidx + 1) * T] = mul(small, big, ell, d)
        big = mul(big, step, ell, d)
    return out[:n]


def quad_coeffs(z_even: np.ndarray, ell: int, d: int):
    """Lagrange weights at an even point (grvec.py:151-161)."""
    m = mask_of(ell)
    z = np.asarray(z_even, dtype=U).reshape(1, d)
    if np.any(z & U(1)):
        raise ValueError("even evaluation point required")
    u = z >> U(1)
    one, two = const(1, ell, d), const(2, ell, d)
    with np.errstate(over="ignore"):
        l0 = mul((z - one) & m, (u - one) & m, ell, d)
        l1 = mul(z, (two - z) & m, ell, d)
        l2 = mul(u, (z - one) & m, ell, d)
    return l0, l1, l2
