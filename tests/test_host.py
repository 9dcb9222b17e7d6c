"""Host-side logic that needs no GPU: the C ABI library loads and exports
every declared symbol, transcript/accounting rules, adversary specs, the
cost model, ring moduli, and the multi-process (gloo) sharding plan."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT


def test_library_exports_every_declared_symbol():
    import ctypes
    from paper_2411_09287_b200 import _lib
    lib = _lib.load()
    hdr = open(os.path.join(ROOT, "include", "r3b200.h")).read()
    declared = set(re.findall(r"^\w[\w\s\*]*?\b(r3_\w+)\(", hdr, re.M))
    assert declared == set(_lib.exported_symbols())
    for name in declared:
        assert isinstance(getattr(lib, name), ctypes._CFuncPtr)
    assert lib.r3_abi_version() == 1


def test_aes_key_expansion_fips197():
    # FIPS-197 appendix A.1 key schedule: last round key word
    import ctypes as C
    from paper_2411_09287_b200 import _lib
    key = bytes.fromhex("2b7e151628aed2a6abf7158809cf4f3c")
    rk = (C.c_uint32 * 44)()
    _lib.load().r3_aes128_expand(key, rk)
    assert [rk[i] for i in (0, 4, 43)] == [0x2b7e1516, 0xa0fafe17, 0xb6630ca6]


def test_transcript_counting_and_csv():
    from paper_2411_09287_b200.transport import Phase, Transcript
    t = Transcript(keep_messages=True)
    t.add(1, 2, Phase.ONLINE, "payload", 8, "x")
    t.add(1, 2, Phase.ONLINE, "digest", 32, "h:x")
    t.bump_round(Phase.ONLINE)
    assert t.bytes_sent(frm=1, to=2, phase=Phase.ONLINE) == 8
    assert t.total_bytes(Phase.ONLINE) == 40
    lines = t.to_csv().splitlines()
    assert lines[0] == "from,to,phase,bytes,rounds"
    assert "P1,P2,online,40,1" in lines


def test_router_rules_coop():
    from paper_2411_09287_b200.transport import CoopRouter, HarnessError, Phase, Transcript
    r = CoopRouter(Transcript())
    with pytest.raises(HarnessError):
        r.send(1, 1, Phase.PRE, "x", b"", count_bytes=0)
    with pytest.raises(HarnessError):
        r.send(1, 2, Phase.ONLINE, "x", b"", count_bytes=0)
    r.send(1, 2, Phase.PRE, "a", b"12345678")
    with pytest.raises(HarnessError):
        r.recv(2, 1, "b")


def test_adversary_spec_parse():
    from paper_2411_09287_b200.transport import AdversaryConfig, Injection
    adv = AdversaryConfig.parse("P0:gamma:+1")
    assert adv.corrupted == 0 and adv.injections[0].site == "gamma" and adv.injections[0].delta == 1
    adv = AdversaryConfig.parse("P2:mz:0x10:7:3")
    assert (adv.corrupted, adv.injections[0].gate, adv.injections[0].lane) == (2, 7, 3)
    with pytest.raises(ValueError):
        AdversaryConfig.parse("P9:gamma:+1")
    inj = Injection("gamma", 1)
    assert inj.matches("dot.gamma", 3) and not inj.matches("vfy.dot.gamma", 3)
    assert Injection("vfy.dot.gamma", 1).matches("vfy.dot.gamma", None)


def test_cost_model_and_pick_r():
    from paper_2411_09287_b200 import verify
    assert verify.online_bits(1024, 7, 64, 64) == (5 * 7 + 3 + 8) * 64 * 64
    assert verify.rounds(5) == 7
    assert verify.pick_r(1, 64, 64) == 0
    assert 0 <= verify.pick_r(64, 64, 64, "lan") <= 6
    assert verify.pick_r(2 ** 20, 64, 64, "wan") >= 7
    assert verify.latency_estimate(1, 0, "lan") == pytest.approx(0.2)
    assert verify.latency_estimate(0, 8e6, "wan") == pytest.approx(200.0)


def test_moduli_and_reduction_rows():
    from paper_2411_09287_b200.rings import ConfigError, RingElem, gf2_is_irreducible, modulus_for_degree
    for d in (1, 2, 4, 8, 16, 32, 64):
        mod = modulus_for_degree(d)
        assert gf2_is_irreducible(mod.f_bits)
        if d > 1:
            rows = mod.reduction_rows(64)
            assert rows.shape == (d - 1, d)
    assert not gf2_is_irreducible(0b101)  # x^2 + 1 = (x+1)^2
    with pytest.raises(ConfigError):
        modulus_for_degree(3)
    assert RingElem(0x8000, 16).sar(4).value == 0xF800
    assert RingElem(5, 4).signed() == 5 and RingElem(15, 4).signed() == -1


def test_reduction_rows_match_oracle_reduction():
    """x^(d+i) mod f from the host table equals the oracle's top-down reduction."""
    from oracle import gr
    from paper_2411_09287_b200.rings import modulus_for_degree
    for d in (8, 16, 64):
        rows = modulus_for_degree(d).reduction_rows(64)
        for i in (0, 1, d - 2):
            xi = np.zeros((1, d), dtype=np.uint64)
            xi[0, 1] = 1                      # x
            xp = np.zeros((1, d), dtype=np.uint64)
            xp[0, d - 1] = 1                  # x^(d-1)
            p = gr.mul(xp, xi, 64, d)         # x^d
            for _ in range(i):
                p = gr.mul(p, xi, 64, d)
            np.testing.assert_array_equal(p[0], rows[i])


def test_coop_scheduler_order_barriers_and_deadlock():
    """The cooperative engine on CPU tensors: a message ring with round
    barriers completes in the reference's round-robin order (global message
    log P0 first), a Session.joint rendezvous hands every party its own
    result, and a program where every party first waits on a message is a
    deadlock (HarnessError), not a hang."""
    import torch
    from paper_2411_09287_b200.runtime import Session
    from paper_2411_09287_b200.sharing import Ring
    from paper_2411_09287_b200.transport import HarnessError
    ring = Ring(64)

    def ring_prog(party):
        nxt, prv = (party.role + 1) % 3, (party.role + 2) % 3
        got = []
        for k in range(4):
            party.send(nxt, f"t{k}", torch.full((2,), 10 * party.role + k, dtype=torch.int64), ring)
            got.append(int(party.recv(prv, f"t{k}", ring, 2)[0]))
            party.round_barrier()
        joint = party.sess.joint(("sum", 0), party.role, party.role + 1,
                                 lambda ins: {r: sum(ins.values()) * 100 + r for r in ins})
        return got, joint

    sess = Session(seed=1, keep_messages=True)
    res = sess.run(ring_prog)
    assert [r[0] for r in res] == [[20, 21, 22, 23], [0, 1, 2, 3], [10, 11, 12, 13]]
    assert [r[1] for r in res] == [600, 601, 602]
    assert [m[0] for m in sess.transcript.messages[:3]] == [0, 1, 2]
    assert sess.transcript.rounds[next(iter(sess.transcript.rounds))] == 4

    def dead(party):
        return party.recv((party.role + 1) % 3, "x", ring, 1)

    with pytest.raises(HarnessError):
        Session(seed=1).run(dead)


def test_deferred_checks_refused_with_adversary():
    """Digest checks of a session with an adversary must be eager (abort
    points and the public-value cache key depend on it)."""
    from paper_2411_09287_b200.rings import ConfigError
    from paper_2411_09287_b200.runtime import Session
    from paper_2411_09287_b200.transport import AdversaryConfig, Injection
    adv = AdversaryConfig(corrupted=1, injections=[Injection("mz", delta=1, gate=0, lane=0)])
    with pytest.raises(ConfigError):
        Session(seed=1, adversary=adv, checks="deferred")
    assert Session(seed=1, adversary=adv).eager_checks
    assert not Session(seed=1).eager_checks


def test_ring3pc_import_path_is_the_b200_package():
    """pkg/src/ring3pc: `import ring3pc` (the reference's import path)
    resolves every reference submodule to the B200 implementation."""
    import importlib
    import sys
    src = os.path.join(ROOT, "pkg", "src")
    sys.path.insert(0, src)
    try:
        for k in [k for k in sys.modules if k == "ring3pc" or k.startswith("ring3pc.")]:
            del sys.modules[k]
        r = importlib.import_module("ring3pc")
        assert r.__file__.startswith(src)
        import paper_2411_09287_b200 as impl
        for name in r.SUBMODULES:
            mod = importlib.import_module(f"ring3pc.{name}")
            assert mod is importlib.import_module(f"paper_2411_09287_b200.{name}")
        from ring3pc.runtime import Session
        assert Session is impl.Session and r.Phase is impl.Phase
    finally:
        sys.path.remove(src)
        for k in [k for k in sys.modules if k == "ring3pc" or k.startswith("ring3pc.")]:
            del sys.modules[k]
