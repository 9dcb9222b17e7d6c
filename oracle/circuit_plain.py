"""Plaintext evaluation of the text circuit format -- TEST INFRASTRUCTURE ONLY.

The cleartext meaning of every gate of the reference's circuit language
(circuit.py:1-20): ring arithmetic mod 2^ell, TRUNC as the arithmetic right
shift, RELU / MAXPOOL on the two's-complement reading.  Works on numpy
object arrays so one call evaluates B independent input assignments.  The
secure evaluator's TRUNC is probabilistic (one ulp), so plain_eval_bounds
also carries a per-lane error bound through the circuit; gates outside a
truncation lineage have bound 0 (exact).
Pinned against the reference's own golden runs in tests/test_circuit_host.py.
"""

from __future__ import annotations

import numpy as np


def _signed(v, ell):
    return np.where(v >> (ell - 1) != 0, v - (1 << ell), v)


def plain_eval(text: str, values: dict, ell: int = 64, lanes: int = 1) -> list[np.ndarray]:
    """values: wire -> int or length-`lanes` sequence.  Returns one object
    array (uint ell-bit values) per OUTPUT line."""
    return plain_eval_bounds(text, values, ell, lanes)[0]


def plain_eval_bounds(text: str, values: dict, ell: int = 64, lanes: int = 1):
    """plain_eval plus, per output, a per-lane bound on how far the secure
    result may sit from it: every probabilistic TRUNC adds one ulp after
    dividing the incoming error by 2^t, products scale an operand's error by
    the other operand's magnitude, RELU / MAXPOOL are 1-Lipschitz."""
    mask = (1 << ell) - 1
    w: dict[int, np.ndarray] = {}
    e: dict[int, np.ndarray] = {}
    outs, errs = [], []
    zero = lambda: np.zeros(lanes, dtype=object)
    mag = lambda i: np.abs(_signed(w[i], ell)) + e[i]

    def val(v):
        arr = np.array([int(x) for x in np.atleast_1d(np.asarray(v, dtype=object))], dtype=object)
        return (np.full(lanes, arr[0], dtype=object) if arr.size == 1 else arr) & mask

    for raw in text.splitlines():
        t = raw.split("#", 1)[0].split()
        if not t:
            continue
        op, ids = t[0].upper(), t[1:]
        if op == "OUTPUT":
            outs.append(w[int(ids[0])].copy())
            errs.append(e[int(ids[0])].copy())
            continue
        dst = int(ids[0])
        src = [int(x, 0) for x in ids[1:]]
        if op in ("ADD", "SUB"):
            e[dst] = e[src[0]] + e[src[1]]
        elif op == "MUL":
            e[dst] = mag(src[0]) * e[src[1]] + mag(src[1]) * e[src[0]]
        elif op == "SCALE":
            c = _signed(np.array([int(ids[1], 0) & mask], dtype=object), ell)[0]
            e[dst] = abs(c) * e[src[1]]
        elif op == "DOT":
            n = src[0]
            acc = zero()
            for a, b in zip(src[1:1 + n], src[1 + n:1 + 2 * n]):
                acc = acc + mag(a) * e[b] + mag(b) * e[a]
            e[dst] = acc
        elif op == "TRUNC":
            e[dst] = (e[src[0]] >> src[1]) + 1 + (e[src[0]] % (1 << src[1]) != 0)
        elif op == "RELU":
            e[dst] = e[src[0]]
        elif op == "MAXPOOL":
            e[dst] = np.max(np.stack([e[x] for x in src[1:1 + src[0]]]), axis=0)
        else:
            e[dst] = zero()
        if op == "INPUT":
            w[dst] = val(values.get(dst, 0))
        elif op == "CONST":
            w[dst] = val(int(ids[1], 0))
        elif op in ("ADD", "SUB", "MUL"):
            a, b = w[int(ids[1])], w[int(ids[2])]
            w[dst] = {"ADD": a + b, "SUB": a - b, "MUL": a * b}[op] & mask
        elif op == "SCALE":
            w[dst] = (int(ids[1], 0) * w[int(ids[2])]) & mask
        elif op == "DOT":
            n = int(ids[1])
            src = [int(x) for x in ids[2:2 + 2 * n]]
            acc = np.zeros(lanes, dtype=object)
            for a, b in zip(src[:n], src[n:]):
                acc = acc + w[a] * w[b]
            w[dst] = acc & mask
        elif op == "TRUNC":
            w[dst] = (_signed(w[int(ids[1])], ell) >> int(ids[2])) & mask
        elif op == "RELU":
            v = w[int(ids[1])]
            w[dst] = np.where(v >> (ell - 1) != 0, 0, v).astype(object)
        elif op == "MAXPOOL":
            n = int(ids[1])
            stack = np.stack([_signed(w[int(x)], ell) for x in ids[2:2 + n]])
            w[dst] = np.max(stack, axis=0).astype(object) & mask
        else:
            raise ValueError(f"unknown op {op}")
    return outs, errs


def ulp_distance(a, b, ell: int = 64) -> int:
    """Largest two's-complement distance between two result arrays."""
    a = _signed(np.asarray(a, dtype=object) & ((1 << ell) - 1), ell)
    b = _signed(np.asarray(b, dtype=object) & ((1 << ell) - 1), ell)
    return int(np.max(np.abs(a - b))) if a.size else 0

