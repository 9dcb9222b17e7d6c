"""Parity of the B200 implementation with the live reference's golden runs.

Every case of tests/programs.py was executed by the unmodified reference
(tests/golden/make_golden.py).  Here the same program runs on the GPU through
`paper_2411_09287_b200` and must reproduce, bit for bit: every party's share
components, opened values, verdicts / abort status, transcript counters,
round counts, the ordered message log, and the SHA-256 of every message
payload as sent.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import golden_names, load_golden

pytestmark = pytest.mark.gpu

PKG = "paper_2411_09287_b200"

# golden program (reference primitives, gathered operands) -> the B200 API
# that must reproduce it (GEMM-form linear layers)
GEMM_FORM = {"infer_batch_gathered": "infer_batch"}


def _flatten(role, res, out, prefix, MVal, host):
    if isinstance(res, dict):
        for k, v in res.items():
            _flatten(role, v, out, f"{prefix}.{k}" if prefix else k, MVal, host)
        return
    if isinstance(res, MVal):
        for name, arr in (("m", res.m), ("s1", res.mask.s1), ("s2", res.mask.s2),
                          ("total", res.mask.total)):
            if arr is not None:
                out["arrays"][f"p{role}.{prefix}.{name}"] = host(arr)
        return
    if isinstance(res, (bool, np.bool_)):
        out["scalars"][f"p{role}.{prefix}"] = bool(res)
        return
    if res is None:
        return
    out["arrays"][f"p{role}.{prefix}"] = host(res)


def run_case(name, engine="coop", prog_override=None, joint=True, pkg=PKG):
    import programs
    from paper_2411_09287_b200 import host
    from paper_2411_09287_b200.runtime import Session
    from paper_2411_09287_b200.sharing import MVal, digest, encode_array
    from paper_2411_09287_b200.transport import AbortError, AdversaryConfig, Injection, DIGEST

    meta, arrays = load_golden(name)
    spec = {c[0]: c for c in programs.CASES + programs.SCALE_CASES}
    tspec = {c[0]: c for c in programs.TAMPER_CASES}
    if name in spec:
        _, prog_name, args, kwargs, sess_kw = spec[name]
        inj = None
    else:
        _, prog_name, args, inj, sess_kw = tspec[name]
        kwargs = {}
    # inputs come from the golden file where they were arrays
    args = tuple(arrays[f"arg{i}"] if f"arg{i}" in arrays else a for i, a in enumerate(args))
    # reference-primitive programs whose B200 counterpart is a different API
    prog_override = prog_override or GEMM_FORM.get(prog_name)
    prog = getattr(programs.build(pkg), prog_override or prog_name)
    adv = None
    if inj is not None:
        site, who, delta, gate, lane = inj
        adv = AdversaryConfig(corrupted=who, injections=[Injection(site, delta=delta, gate=gate, lane=lane)])
    sess = Session(seed=sess_kw.get("seed", 0), ell=sess_kw.get("ell", 64), adversary=adv,
                   keep_messages=True, engine=engine, joint=joint)
    log = []

    def hook(frm, to, phase, label, arr, cls, ring):
        enc = encode_array(arr, ring)
        if cls == DIGEST:
            enc = digest(sess.salt, label[2:], enc)
        log.append((frm, to, phase.value, label, cls, hashlib.sha256(enc).hexdigest()))

    sess.message_hook = hook
    out = {"arrays": {}, "scalars": {}}
    status = "ok"
    try:
        res = sess.run(lambda party: prog(party, *args, **kwargs))
        for role in range(3):
            _flatten(role, res[role], out, "", MVal, host)
    except AbortError as e:
        status = f"abort:P{e.party}"
    return meta, arrays, sess, log, out, status


def _per_sender(msgs):
    by = {}
    for m in msgs:
        by.setdefault(m[0], []).append(tuple(m))
    return by


@pytest.mark.parametrize("name", golden_names())
def test_golden_case(cuda, name):
    meta, arrays, sess, log, out, status = run_case(name)
    assert status == meta["status"]
    tr = sess.transcript
    counters = sorted([[f, t, p.value, c, n] for (f, t, p, c), n in tr.counters.items()])
    assert counters == meta["counters"]
    assert {p.value: n for p, n in tr.rounds.items()} == meta["rounds"]
    msgs = [[f, t, p.value, lab, nb, c] for (f, t, p, lab, nb, c) in tr.messages]
    assert _per_sender(msgs) == _per_sender(meta["messages"])
    assert _per_sender(log) == _per_sender([tuple(x) for x in meta["payloads"]])
    assert out["scalars"] == meta["scalars"]
    want = {k: v for k, v in arrays.items() if not k.startswith("arg")}
    assert sorted(out["arrays"]) == sorted(want)
    for k, v in want.items():
        np.testing.assert_array_equal(out["arrays"][k].reshape(v.shape), v, err_msg=k)


@pytest.mark.parametrize("name", ["mulv_64_d16_R2", "relu_64"])
def test_golden_coop_message_order(cuda, name):
    """With gate-by-gate scheduling (joint=False) the coop engine reproduces
    the reference's global message order; joint kernels (the default) keep
    every per-sender sequence (test_golden_case) but interleave differently."""
    meta, _a, sess, _l, _o, _s = run_case(name, joint=False)
    msgs = [[f, t, p.value, lab, nb, c] for (f, t, p, lab, nb, c) in sess.transcript.messages]
    assert msgs == meta["messages"]


@pytest.mark.parametrize("name", ["relu_64", "infer1_conv_tiny", "mulv_1024_d64_R7"])
def test_golden_without_joint_kernels(cuda, name):
    """The gate-by-gate path (joint=False) matches the same golden runs."""
    meta, arrays, sess, log, out, status = run_case(name, joint=False)
    assert status == meta["status"]
    assert _per_sender(log) == _per_sender([tuple(x) for x in meta["payloads"]])
    want = {k: v for k, v in arrays.items() if not k.startswith("arg")}
    for k, v in want.items():
        np.testing.assert_array_equal(out["arrays"][k].reshape(v.shape), v, err_msg=k)


def test_golden_threads_engine(cuda):
    meta, arrays, sess, _l, out, status = run_case("mulv_100_d64_R3", engine="threads")
    assert status == "ok"
    assert out["scalars"] == meta["scalars"]
    np.testing.assert_array_equal(out["arrays"]["p1.z.m"], arrays["p1.z.m"])


@pytest.mark.parametrize("name", ["matmul_8x8x8", "matmul_12x16x10"])
def test_matmul_gemm_form_matches_gathered_golden(cuda, name):
    """gates.matmul_prepare/finish (tensor-core GEMMs) reproduce the
    reference's gathered Pi_dot linear layer bit for bit."""
    meta, arrays, sess, log, out, status = run_case(name, prog_override="matmul_gemm")
    assert status == meta["status"]
    counters = sorted([[f, t, p.value, c, n] for (f, t, p, c), n in sess.transcript.counters.items()])
    assert counters == meta["counters"]
    assert _per_sender(log) == _per_sender([tuple(x) for x in meta["payloads"]])
    want = {k: v for k, v in arrays.items() if not k.startswith("arg")}
    for k, v in want.items():
        np.testing.assert_array_equal(out["arrays"][k].reshape(v.shape), v, err_msg=k)


@pytest.mark.parametrize("name", ["mulv_1024_d64_R7", "relu_64", "infer1_mlp_tiny"])
def test_golden_through_ring3pc_import_path(cuda, name):
    """Unmodified reference-shaped programs written against `ring3pc`
    (tests/programs.py builds them from `ring3pc.gates`, `ring3pc.verify`,
    ...) run on the GPU through pkg/src/ring3pc and match the reference."""
    import os
    import sys
    from conftest import ROOT
    src = os.path.join(ROOT, "pkg", "src")
    sys.path.insert(0, src)
    try:
        for k in [k for k in sys.modules if k == "ring3pc" or k.startswith("ring3pc.")]:
            del sys.modules[k]
        import ring3pc
        assert ring3pc.__file__.startswith(src)
        meta, arrays, sess, log, out, status = run_case(name, pkg="ring3pc")
    finally:
        sys.path.remove(src)
        for k in [k for k in sys.modules if k == "ring3pc" or k.startswith("ring3pc.")]:
            del sys.modules[k]
    assert status == meta["status"]
    assert _per_sender(log) == _per_sender([tuple(x) for x in meta["payloads"]])
    want = {k: v for k, v in arrays.items() if not k.startswith("arg")}
    for k, v in want.items():
        np.testing.assert_array_equal(out["arrays"][k].reshape(v.shape), v, err_msg=k)
