"""Bit-exact parity at config-relevant sizes.

The cases of tests/programs.py:SCALE_CASES were run by the unmodified
reference (tests/golden/make_golden.py --scale, tens of seconds each on the
CPU).  Their fixtures keep a SHA-256 per output array (every party's share
components, opened values) plus the full transcript: counters, rounds, the
per-sender message log and the SHA-256 of every message payload.  Here the
same programs run on the GPU and every digest must match.

Sizes are chosen so the multi-stage pipelines wrap: the d = 64 tensor-core
base fold (bf_tc.cu) runs several 32-block K-steps per CTA at N = 2^16, the
joint d = 16 level folds (lf16_tc.cu) see >= 2^14 dense rows inside a
verified ReLU of 4096 lanes, and the factorised Pi_bsv of a verified
matmul runs six structured levels before materialising.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import scale_golden_names
from test_gpu_golden import GEMM_FORM, _per_sender, run_case

pytestmark = pytest.mark.gpu


def array_digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u8").tobytes()).hexdigest()


def _check(meta, sess, log, out, status):
    assert status == meta["status"]
    tr = sess.transcript
    counters = sorted([[f, t, p.value, c, n] for (f, t, p, c), n in tr.counters.items()])
    assert counters == meta["counters"]
    assert {p.value: n for p, n in tr.rounds.items()} == meta["rounds"]
    msgs = [[f, t, p.value, lab, nb, c] for (f, t, p, lab, nb, c) in tr.messages]
    assert _per_sender(msgs) == _per_sender(meta["messages"])
    assert _per_sender(log) == _per_sender([tuple(x) for x in meta["payloads"]])
    assert out["scalars"] == meta["scalars"]
    want = meta["array_sha256"]
    assert sorted(out["arrays"]) == sorted(want)
    for k, (h, shape) in want.items():
        got = np.asarray(out["arrays"][k]).reshape(shape)
        assert array_digest(got) == h, k


@pytest.mark.parametrize("name", scale_golden_names())
def test_scale_golden(cuda, name):
    import programs
    prog = {c[0]: c[1] for c in programs.SCALE_CASES}[name]
    override = "matmul_gemm" if prog == "matmul" else GEMM_FORM.get(prog)
    meta, _arrays, sess, log, out, status = run_case(name, prog_override=override)
    _check(meta, sess, log, out, status)


@pytest.mark.parametrize("name", ["relu_4096_d16_auto"])
def test_scale_golden_gate_by_gate(cuda, name):
    """The same case with joint kernels off (per-party launches)."""
    meta, _arrays, sess, log, out, status = run_case(name, joint=False)
    assert status == meta["status"]
    assert _per_sender(log) == _per_sender([tuple(x) for x in meta["payloads"]])
    for k, (h, shape) in meta["array_sha256"].items():
        assert array_digest(np.asarray(out["arrays"][k]).reshape(shape)) == h, k


def test_scale_golden_matmul_gathered(cuda):
    """The verified matmul case through the reference-shaped gathered Pi_dot
    (dense Pi_bsv path) as well as the GEMM form above."""
    meta, _arrays, sess, log, out, status = run_case("matmul_v_24x64x40")
    _check(meta, sess, log, out, status)
