"""Parity at bench sizes through size-independent properties (SURVEY 8c:
the live reference cannot run these sizes): verdicts, opened results equal
to the plaintext computation, tamper -> abort, and random-lane spot checks
of shares against the seekable AES-CTR restatement (oracle/prf.py)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _mulv_prog(N, d, R, ring_ell=64):
    from paper_2411_09287_b200 import gates, verify
    from paper_2411_09287_b200.sharing import Ring, shc_random
    from paper_2411_09287_b200.transport import Phase

    def prog(party):
        ring = Ring(ring_ell)
        party.enter_phase(Phase.PRE)
        x = shc_random(party, N, ring)
        y = shc_random(party, N, ring)
        g = gates.mul_prepare(party, x.mask, y.mask, N)
        verify.prepare_verification(party, d=d, r_max=max(R, 1))
        party.round_barrier()
        party.enter_phase(Phase.ONLINE)
        z = gates.mul_finish(party, g, x, y)
        party.round_barrier()
        party.enter_phase(Phase.POST)
        return x, y, z, verify.batch_verify_muls(party, ring_ell, d=d, R=R)
    return prog


def test_mulv_2_22_products_verdict_and_prf_spot_checks(cuda):
    """N = 2^22, d = 64, R = pick_r: honest verdict, z = x y for every lane,
    and sampled mask shares equal the AES-CTR stream words the reference's
    Prg would draw (P1's x.s1 = first N words of ("01", "sha"), masked)."""
    from oracle import prf as oprf
    from paper_2411_09287_b200 import host, verify
    from paper_2411_09287_b200.runtime import Session
    from paper_2411_09287_b200.sharing import reconstruct_clear
    N, d = 1 << 22, 64
    R = verify.pick_r(N, 64, d)
    seed = 12345
    res = Session(seed=seed).run(_mulv_prog(N, d, R))
    assert all(r[3] for r in res)
    x = host(reconstruct_clear([r[0] for r in res]))
    y = host(reconstruct_clear([r[1] for r in res]))
    z = host(reconstruct_clear([r[2] for r in res]))
    with np.errstate(over="ignore"):
        np.testing.assert_array_equal(z, x * y)
    seeds = oprf.pair_seeds(seed.to_bytes(16, "little"))
    key01 = oprf.stream_key(seeds["01"], "sha")
    s1 = host(res[1][0].mask.s1)
    for lane in np.random.default_rng(0).integers(0, N, 16):
        assert int(s1[lane]) == int(oprf.keystream(key01, int(lane), 1)[0])
    # y's s1 follows x's on the same stream (shc_random draws x then y)
    ys1 = host(res[1][1].mask.s1)
    for lane in (0, N - 1, N // 3):
        assert int(ys1[lane]) == int(oprf.keystream(key01, N + lane, 1)[0])


def test_mulv_tamper_at_scale_aborts(cuda):
    """An additive attack on one lane's online message of a 2^20 batch is
    caught by the batch check (d = 64, R = pick_r)."""
    from paper_2411_09287_b200 import verify
    from paper_2411_09287_b200.runtime import Session
    from paper_2411_09287_b200.transport import AbortError, AdversaryConfig, Injection
    N, d = 1 << 20, 64
    R = verify.pick_r(N, 64, d)
    adv = AdversaryConfig(corrupted=1, injections=[Injection("dot.mz", delta=1, gate=0, lane=777)])
    try:
        res = Session(seed=7, adversary=adv).run(_mulv_prog(N, d, R))
    except AbortError:
        return
    assert not all(r[3] for r in res), "tampered multiplication verified"


def test_relu_2_18_matches_plaintext(cuda):
    """Secure ReLU over 2^18 fixed-point inputs with verify_session (d = 16,
    R auto) opens exactly max(x, 0)."""
    import torch
    import bench
    from paper_2411_09287_b200.runtime import Session
    N = 1 << 18
    xv = np.trunc(np.random.default_rng(4).normal(0, 4, N) * 2 ** 16).astype(np.int64)
    prog = bench.make_relu_program(N, 16)
    out = Session(seed=3).run(prog, torch.from_numpy(xv), True)[0]
    np.testing.assert_array_equal(out.cpu().numpy(), np.where(xv >= 0, xv, 0))


def _matmul_prog(n, X, W, check):
    import torch
    from paper_2411_09287_b200 import gates, verify
    from paper_2411_09287_b200.sharing import Ring, rec, shc_input_mask, shc_input_online
    from paper_2411_09287_b200.transport import Phase

    def prog(party):
        ring = Ring(64)
        party.enter_phase(Phase.PRE)
        xm = shc_input_mask(party, 2, n * n, ring)
        wm = shc_input_mask(party, 1, n * n, ring)
        tr = gates.trunc_prepare(party, n * n, 16, ring)
        g = gates.matmul_prepare(party, xm, wm, n, n, n, out_mask=tr.rx_mask)
        if check:
            verify.prepare_verification(party, d=16)
        party.round_barrier()
        party.enter_phase(Phase.ONLINE)
        Xs = shc_input_online(party, 2, torch.from_numpy(X.reshape(-1)) if party.role == 2 else None, xm,
                              n * n, ring, "X")
        Ws = shc_input_online(party, 1, torch.from_numpy(W.reshape(-1)) if party.role == 1 else None, wm,
                              n * n, ring, "W")
        z = gates.trunc_online(party, gates.matmul_finish(party, g, Xs, Ws, log=check), tr)
        party.round_barrier()
        party.enter_phase(Phase.POST)
        verdict = None
        if check:
            verdict = verify.verify_session(party, d=16, R="auto")
            if not all(verdict.values()):
                party.abort("verification failed")   # ppml.py:440-445: never open after a failed check
        else:
            party.freeze_logs()
        return rec(party, z, "z").cpu().numpy(), verdict
    return prog


@pytest.mark.parametrize("check", [False, True])
def test_matmul_512_trunc_against_plaintext(cuda, check):
    """Share matmul 512^3 + probabilistic truncation (t = 16): every opened
    entry is within one ulp of floor(X W / 2^16) (gates.py:248-302); with
    check=True the GEMM-form dot log (factorised Pi_bsv, nine structured
    levels) and the truncation bit dots are verified first and accepted."""
    from paper_2411_09287_b200.runtime import Session
    n = 512
    rng = np.random.default_rng(9)
    X = np.trunc(rng.normal(0, 1, (n, n)) * 2 ** 16).astype(np.int64)
    W = np.trunc(rng.normal(0, 1 / 16, (n, n)) * 2 ** 16).astype(np.int64)
    got, verdict = Session(seed=2).run(_matmul_prog(n, X, W, check))[0]
    if check:
        assert verdict and all(verdict.values()), verdict
    exact = X.astype(object).dot(W.astype(object))
    want = np.vectorize(lambda v: int(v) >> 16, otypes=[object])(exact)
    diff = np.abs(got.reshape(n, n).astype(object) - want)
    assert int(diff.max()) <= 1


@pytest.mark.parametrize("site,who", [("mz", 1), ("z", 2), ("gamma", 0)])
def test_matmul_512_verified_tamper_aborts(cuda, site, who):
    """One tampered lane in the 512^3 share matmul (the P1 -> P2 leg, a
    party's local output share, or P0's Gamma deal of the GEMM gate) is
    caught by the verified session: run() raises AbortError."""
    from paper_2411_09287_b200.runtime import Session
    from paper_2411_09287_b200.transport import AbortError, AdversaryConfig, Injection
    n = 512
    rng = np.random.default_rng(10)
    X = np.trunc(rng.normal(0, 1, (n, n)) * 2 ** 16).astype(np.int64)
    W = np.trunc(rng.normal(0, 1 / 16, (n, n)) * 2 ** 16).astype(np.int64)
    # gate ids of kind "dot": the truncation's two bit dots are dealt first
    # (trunc_prepare), then the GEMM gate
    adv = AdversaryConfig(corrupted=who, injections=[Injection(site, delta=1, gate=2, lane=12345)])
    with pytest.raises(AbortError):
        Session(seed=3, adversary=adv).run(_matmul_prog(n, X, W, True))


@pytest.mark.parametrize("n,lanes,d", [(64, 1 << 16, 16), (4, 1 << 18, 64)])
def test_dot_log_at_scale_verdicts(cuda, n, lanes, d):
    """Pi_bsv over a large dot log (the ReLU's n = 64 edaBits dots at d = 16,
    short dots at d = 64; R = pick_r): the honest run verifies and opens
    sum_k x_k y_k on every lane, and an additive error on one lane's leg of
    the same log is caught."""
    import programs
    from paper_2411_09287_b200 import host, verify
    from paper_2411_09287_b200.runtime import Session
    from paper_2411_09287_b200.sharing import reconstruct_clear
    from paper_2411_09287_b200.transport import AbortError, AdversaryConfig, Injection
    R = verify.pick_r(n * lanes, 64, d)
    prog = programs.build("paper_2411_09287_b200").dotv
    res = Session(seed=5).run(prog, n, lanes, d, R)
    assert all(r["verdict"]["dot"] for r in res)
    z = host(reconstruct_clear([r["z"] for r in res]))
    assert z.shape == (lanes,)
    adv = AdversaryConfig(corrupted=1, injections=[Injection("dot.mz", delta=3, gate=0, lane=lanes // 3)])
    try:
        res = Session(seed=5, adversary=adv).run(prog, n, lanes, d, R)
    except AbortError:
        return
    assert not all(r["verdict"]["dot"] for r in res), "tampered dot log verified"


def test_mulv_d16_at_scale_honest_and_tamper(cuda):
    """d = 16 multiplication logs large enough for the tensor-core base fold
    (2^20 gates): the honest run verifies with z = x y, one tampered leg is
    caught."""
    from paper_2411_09287_b200 import host, verify
    from paper_2411_09287_b200.runtime import Session
    from paper_2411_09287_b200.sharing import reconstruct_clear
    from paper_2411_09287_b200.transport import AbortError, AdversaryConfig, Injection
    N, d = 1 << 20, 16
    R = verify.pick_r(N, 64, d)
    res = Session(seed=21).run(_mulv_prog(N, d, R))
    assert all(r[3] for r in res)
    x = host(reconstruct_clear([r[0] for r in res]))
    y = host(reconstruct_clear([r[1] for r in res]))
    z = host(reconstruct_clear([r[2] for r in res]))
    with np.errstate(over="ignore"):
        np.testing.assert_array_equal(z, x * y)
    adv = AdversaryConfig(corrupted=2, injections=[Injection("dot.mz", delta=1 << 40, gate=0, lane=12345)])
    try:
        res = Session(seed=21, adversary=adv).run(_mulv_prog(N, d, R))
    except AbortError:
        return
    assert not all(r[3] for r in res), "tampered d = 16 multiplication verified"
