"""Session-level behaviour on the GPU: deferred digest checks abort a run
whose openings disagree, and per-run state does not leak between runs."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _mul_open_program():
    from paper_2411_09287_b200 import gates
    from paper_2411_09287_b200.sharing import Ring, rec, shc_input
    from paper_2411_09287_b200.transport import Phase

    def prog(party):
        ring = Ring(64)
        party.enter_phase(Phase.PRE)
        party.enter_phase(Phase.ONLINE)
        x = shc_input(party, 0, np.array([3, 5], np.uint64) if party.role == 0 else None, 2, ring, "x")
        y = shc_input(party, 1, np.array([4, 6], np.uint64) if party.role == 1 else None, 2, ring, "y")
        z = gates.mul(party, x, y)
        party.round_barrier()
        party.enter_phase(Phase.POST)
        party.freeze_logs()
        return rec(party, z, "z")
    return prog


def test_deferred_digest_mismatch_aborts(cuda):
    """A payload altered in flight on an honest (deferred-check) session:
    the mismatch is only counted on the device during the run, and run()
    raises AbortError when it settles the counter."""
    from paper_2411_09287_b200.runtime import Session
    from paper_2411_09287_b200.transport import AbortError, CoopRouter

    class Tamper(CoopRouter):
        done = False

        def send(self, frm, to, phase, label, payload, cls="payload", count_bytes=None):
            if label.startswith("h:") and not Tamper.done and hasattr(payload, "add_"):
                payload = payload.clone()
                payload.view(-1)[0] += 1
                Tamper.done = True
            return super().send(frm, to, phase, label, payload, cls, count_bytes)

    sess = Session(seed=5, router_cls=Tamper)
    assert not sess.eager_checks
    with pytest.raises(AbortError):
        sess.run(_mul_open_program())
    assert Tamper.done
    assert sess._deferred is None and sess._deferred_what == [] and sess._deferred_small == []
    ok = Session(seed=5).run(_mul_open_program())
    assert [int(v) for v in ok[0].cpu()] == [12, 30]


def test_session_rerun_after_discarded_logs(cuda):
    """A Session that ran an unverified program with discarded logs can run
    a verified program afterwards (discard is scoped to one run)."""
    from paper_2411_09287_b200 import gates, verify
    from paper_2411_09287_b200.runtime import Session
    from paper_2411_09287_b200.sharing import Ring, shc_random
    from paper_2411_09287_b200.transport import Phase

    def unverified(party):
        party.discard_logs()
        return True

    def verified(party):
        ring = Ring(64)
        party.enter_phase(Phase.PRE)
        x = shc_random(party, 64, ring)
        y = shc_random(party, 64, ring)
        g = gates.mul_prepare(party, x.mask, y.mask, 64)
        verify.prepare_verification(party, d=16, r_max=2)
        party.round_barrier()
        party.enter_phase(Phase.ONLINE)
        gates.mul_finish(party, g, x, y)
        party.round_barrier()
        party.enter_phase(Phase.POST)
        return verify.batch_verify_muls(party, 64, d=16, R=2)

    sess = Session(seed=9)
    sess.run(unverified)
    assert all(p.logs[k].discard for p in sess.parties for k in p.logs)
    assert all(Session(seed=9).run(verified))


@pytest.mark.parametrize("N,R,d", [((1 << 16) + 5, 5, 64), ((1 << 15) + 3, 3, 64), ((1 << 16) + 5, 5, 16)])
def test_base_reduction_block_sizes_give_identical_transcripts(cuda, N, R, d, monkeypatch):
    """The d = 64 verification of one multiplication log through the
    two-level base reduction (blocks of four, B = 0), three levels from
    the base (B = 8) and four (B = 16, where the log is large enough): every
    message payload (per sender, in order), the verdict and the opened
    product are identical -- the block size only changes how the same
    values are computed (verify.py:168-241).  A tampered leg is still
    rejected under the widest form (per-party launches: adversary sessions
    do not batch the parties)."""
    import hashlib
    from paper_2411_09287_b200 import gates, host, verify
    from paper_2411_09287_b200.runtime import Session
    from paper_2411_09287_b200.sharing import Ring, reconstruct_clear, shc_random
    from paper_2411_09287_b200.transport import Phase

    def prog(party):
        ring = Ring(64)
        party.enter_phase(Phase.PRE)
        x = shc_random(party, N, ring)
        y = shc_random(party, N, ring)
        g = gates.mul_prepare(party, x.mask, y.mask, N)
        verify.prepare_verification(party, d=d, r_max=R)
        party.round_barrier()
        party.enter_phase(Phase.ONLINE)
        z = gates.mul_finish(party, g, x, y)
        party.round_barrier()
        party.enter_phase(Phase.POST)
        return z, verify.batch_verify_muls(party, 64, d=d, R=R)

    orig = verify._base_block
    runs = {}
    for B in (0, 8, 16):
        monkeypatch.setattr(verify, "_base_block",
                            lambda comp, R_, gr, B=B: min(B, orig(comp, R_, gr)) if B else 0)
        sess = Session(seed=11)
        log = []
        sess.message_hook = lambda frm, to, ph, label, arr, cls, ring: log.append(
            (frm, label, hashlib.sha256(host(arr).tobytes()).hexdigest()))
        res = sess.run(prog)
        z = host(reconstruct_clear([r[0] for r in res]))
        runs[B] = (sorted(log), [r[1] for r in res], z)
    for B in (8, 16):
        assert runs[B][1] == runs[0][1] == [True, True, True]
        np.testing.assert_array_equal(runs[B][2], runs[0][2])
        assert runs[B][0] == runs[0][0], f"B = {B}: message payloads differ from the two-level form"
    monkeypatch.setattr(verify, "_base_block", orig)
    from paper_2411_09287_b200.transport import AdversaryConfig, Injection
    adv = AdversaryConfig(corrupted=1, injections=[Injection("dot.mz", delta=1, gate=0, lane=7)])
    res = Session(seed=11, adversary=adv).run(prog)
    assert not any(r[1] for r in res), "a tampered leg passed verification"


@pytest.mark.parametrize("what", ["relu", "lenet"])
def test_lane16_dot_form_gives_identical_transcripts(cuda, what, monkeypatch):
    """Dot logs whose lanes hold a multiple of 16 elements (the edaBits inner
    products) verified through the four-level base form (r3_vfy_lane16_fold /
    _line) and through the two-level form (R3_LANES16=0 equivalent): every
    message payload per sender, the verdicts and the outputs are identical
    -- a whole-log ReLU session (_reduce_lanes16) and a verified LeNet-28
    batch (structured dot verification, _Lane16Batch beside FC / conv
    batches)."""
    import hashlib
    import torch
    from paper_2411_09287_b200 import host, ppml, verify
    from paper_2411_09287_b200.runtime import Session
    import bench

    if what == "relu":
        N = 1 << 12
        xv = np.trunc(np.random.default_rng(3).normal(0, 4, N) * 2 ** 16).astype(np.int64)
        prog, args = bench.make_relu_program(N, 16), (torch.from_numpy(xv), True)
    else:
        model = ppml.lenet28_model(np.random.default_rng(0))
        imgs = np.random.default_rng(1).normal(0, 1, (2, int(np.prod(model.input_shape))))
        prog, args = (lambda p: ppml.infer_batch(p, model, imgs if p.role == 2 else None, ppml.InferConfig(d=16),
                                                 batch=2)), ()
    used = []
    orig_fold = verify._block_fold_weights

    def spy(party, k, ws, B, gr):
        used.append(B)
        return orig_fold(party, k, ws, B, gr)
    runs = {}
    for off in (True, False):
        monkeypatch.setattr(verify, "_LANES16_OFF", off)
        monkeypatch.setattr(verify, "_block_fold_weights", spy)
        used.clear()
        sess = Session(seed=5)
        log = []
        sess.message_hook = lambda frm, to, ph, label, arr, cls, ring: log.append(
            (frm, label, hashlib.sha256(host(arr).tobytes()).hexdigest()))
        res = sess.run(prog, *args)
        runs[off] = (sorted(log), res, bool(used))
    assert runs[False][2], "the lane16 form was not exercised"
    assert runs[False][0] == runs[True][0], "message payloads differ from the two-level form"
    flat = lambda res: [host(t) if isinstance(t, torch.Tensor) else t for t in res]
    assert repr(flat(runs[False][1])) == repr(flat(runs[True][1]))
