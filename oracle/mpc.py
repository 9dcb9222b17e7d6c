"""All-party restatement of the verified-multiplication path -- test
infrastructure only.

The reference runs three party coroutines exchanging messages
(runtime.py:177-241); this oracle computes the three parties' views directly
in one numpy program, in the reference's order of PRF draws, messages and
barriers, and books the transcript the way the reference does.  It follows:

  sharing.py:272-314 (sha_random / sha_input / shc_random)
  sharing.py:364-419 (rec message flows)
  gates.py:41-117    (Pi_dot prepare / finish, P0 cross term, P1/P2 legs)
  verify.py:101-119  (prepare_verification challenge draws)
  verify.py:126-263  (lift, compress, reduce_dimension, check_inner_product)
  verify.py:278-311  (batch_verify_muls driver)

A share is a dict role -> {component: array}; P0 holds s1/s2/total, P1 s1/m,
P2 s2/m (SPEC share layout).  Pinned against tests/golden/ (live reference
runs) in tests/test_oracle.py.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import gr
from .prf import Stream, pair_seeds

U = np.uint64
PRE, ONLINE, POST = "preprocessing", "online", "postprocessing"


def _m(ell):
    return U((1 << ell) - 1)


def _wrap(fn):
    with np.errstate(over="ignore"):
        return fn()


class Sim:
    """Streams, ids, phase, transcript of one simulated session."""

    def __init__(self, seed: int, ell: int = 64):
        self.ell = ell
        self.seeds = pair_seeds(seed.to_bytes(16, "little"))
        self.streams: dict = {}
        self.ids: dict = {}
        self.phase = PRE
        self.counters: dict = {}
        self.rounds = {PRE: 0, ONLINE: 0, POST: 0}
        self.messages: list = []

    def draw(self, pair, domain, lanes, ell, d=1):
        key = (pair, domain)
        if key not in self.streams:
            self.streams[key] = Stream(self.seeds[pair], domain)
        v = self.streams[key].base(lanes * d, ell)
        return v if d == 1 else v.reshape(lanes, d)

    def bits(self, pair, domain, n):
        key = (pair, domain)
        if key not in self.streams:
            self.streams[key] = Stream(self.seeds[pair], domain)
        return self.streams[key].bits(n)

    def next_id(self, kind):
        n = self.ids.get(kind, 0)
        self.ids[kind] = n + 1
        return n

    def send(self, frm, to, label, nwords, ell, cls="payload"):
        nbytes = nwords * math.ceil(ell / 8)
        key = (frm, to, self.phase, cls)
        self.counters[key] = self.counters.get(key, 0) + nbytes
        self.messages.append((frm, to, self.phase, label, nbytes, cls))

    def digest(self, frm, to, label):
        key = (frm, to, self.phase, "digest")
        self.counters[key] = self.counters.get(key, 0) + 32
        self.messages.append((frm, to, self.phase, "h:" + label, 32, "digest"))

    def barrier(self):
        self.rounds[self.phase] += 1

    def rounds_by_phase(self, Phase):
        return {p: self.rounds[p.value] for p in Phase}


# ---------------------------------------------------------------------------
# share generation and opening
# ---------------------------------------------------------------------------

def sha_random(sim, lanes, ell, d=1, domain="sha"):
    s1 = sim.draw("01", domain, lanes, ell, d)
    s2 = sim.draw("02", domain, lanes, ell, d)
    tot = _wrap(lambda: (s1 + s2) & _m(ell))
    return {0: {"s1": s1, "s2": s2, "total": tot}, 1: {"s1": s1}, 2: {"s2": s2}}


def shc_random(sim, lanes, ell, d=1, domain="sha"):
    sh = sha_random(sim, lanes, ell, d, domain)
    m = sim.draw("12", domain + ".m", lanes, ell, d)
    sh[1]["m"] = m
    sh[2]["m"] = m
    return sh


def sha_input(sim, x, lanes, ell, d, tag, cls="payload"):
    s1 = sim.draw("01", "sha", lanes, ell, d)
    s2 = _wrap(lambda: (x - s1) & _m(ell))
    sim.send(0, 2, f"sha.{tag}", lanes * d, ell, cls)
    return {0: {"s1": s1, "s2": s2, "total": x}, 1: {"s1": s1}, 2: {"s2": s2}}


def rec(sim, v, tag, ell, d=1, style="open", p0_halves=True):
    """Verifiable opening: message flow of sharing.py:364-419; value m - r."""
    cls_m = "aux" if style == "aux" else "payload"
    cls_r = "payload" if style == "open" else "aux"
    tag = f"{tag}#{sim.next_id('rec')}"
    lanes = v[1]["m"].shape[0]
    nw = lanes * d
    L = lambda leg: f"rec.{tag}.{leg}"
    if p0_halves:
        sim.send(0, 2, L("r1"), nw, ell, cls_r)
        sim.send(0, 1, L("r2"), nw, ell, cls_r)
        sim.send(1, 0, L("m"), nw, ell, cls_m)
        sim.digest(1, 2, L("r1"))
        sim.digest(2, 0, L("m"))
        sim.digest(2, 1, L("r2"))
    else:
        sim.digest(0, 1, L("rsum"))
        sim.digest(0, 2, L("rsum"))
        sim.send(1, 2, L("r1"), nw, ell, cls_r)
        sim.send(1, 0, L("m"), nw, ell, cls_m)
        sim.send(2, 1, L("r2"), nw, ell, cls_r)
        sim.digest(2, 0, L("m"))
    return _wrap(lambda: (v[1]["m"] - v[1]["s1"] - v[2]["s2"]) & _m(ell))


# ---------------------------------------------------------------------------
# Pi_mul over the base ring (n = 1 inner product)
# ---------------------------------------------------------------------------

def mul_gate(sim, x, y, lanes, ell, kind="dot"):
    """mul_prepare + mul_finish (gates.py:52-117 with n = 1)."""
    m = _m(ell)
    gid = sim.next_id(kind)
    out = sha_random(sim, lanes, ell)
    gam = _wrap(lambda: (x[0]["total"] * y[0]["total"] + out[0]["total"]) & m)
    g = sha_input(sim, gam, lanes, ell, 1, f"{kind}.gamma.{gid}")
    return gid, out, g


def mul_finish(sim, gid, out, g, x, y, lanes, ell, kind="dot"):
    m = _m(ell)
    leg1 = _wrap(lambda: (g[1]["s1"] - x[1]["m"] * y[1]["s1"] - y[1]["m"] * x[1]["s1"]) & m)
    leg2 = _wrap(lambda: (x[2]["m"] * y[2]["m"] + g[2]["s2"] - x[2]["m"] * y[2]["s2"]
                          - y[2]["m"] * x[2]["s2"]) & m)
    sim.send(1, 2, f"{kind}.mz.{gid}.leg1", lanes, ell)
    sim.send(2, 1, f"{kind}.mz.{gid}.leg2", lanes, ell)
    mz = _wrap(lambda: (leg1 + leg2) & m)
    z = {r: dict(out[r]) for r in range(3)}
    z[1]["m"] = mz
    z[2]["m"] = mz
    return z


# ---------------------------------------------------------------------------
# extension-ring machinery for verification
# ---------------------------------------------------------------------------

def _comps(role):
    return ("total",) if role == 0 else (("s1", "m") if role == 1 else ("s2", "m"))


def _sub(a, b, ell):
    return _wrap(lambda: (a - b) & _m(ell))


def _add(a, b, ell):
    return _wrap(lambda: (a + b) & _m(ell))


def gr_dot(sim, F, G, ell, d, kind="vfy.dot", lanes_out=1, leg2_cls="payload", gamma_cls="offline"):
    """_gr_dot (verify.py:154-161): dims (N, d) -> (1, d)."""
    gid = sim.next_id(kind)
    out = sha_random(sim, 1, ell, d)
    cross = gr.dot(F[0]["total"], G[0]["total"], ell, d)
    g = sha_input(sim, _add(cross, out[0]["total"], ell), 1, ell, d, f"{kind}.gamma.{gid}", gamma_cls)
    leg1 = _sub(_sub(g[1]["s1"], gr.dot(F[1]["m"], G[1]["s1"], ell, d), ell),
                gr.dot(G[1]["m"], F[1]["s1"], ell, d), ell)
    leg2 = _sub(_sub(_add(gr.dot(F[2]["m"], G[2]["m"], ell, d), g[2]["s2"], ell),
                     gr.dot(F[2]["m"], G[2]["s2"], ell, d), ell),
                gr.dot(G[2]["m"], F[2]["s2"], ell, d), ell)
    sim.send(1, 2, f"{kind}.mz.{gid}.leg1", d, ell)
    sim.send(2, 1, f"{kind}.mz.{gid}.leg2", d, ell, leg2_cls)
    mz = _add(leg1, leg2, ell)
    res = {r: dict(out[r]) for r in range(3)}
    res[1]["m"] = mz
    res[2]["m"] = mz
    return res


def _map(v, fn):
    return {r: {k: fn(a) for k, a in v[r].items()} for r in range(3)}


def _zip(v, w, fn):
    return {r: {k: fn(v[r][k], w[r][k]) for k in v[r] if k in w[r]} for r in range(3)}


def _scale_gr(v, c, ell, d):
    return _map(v, lambda a: gr.mul(a, c, ell, d))


def reduce_dimension(sim, xs, ys, z, ell, d, zeta):
    """verify.py:215-241 (h(1), h(2) by inner products, h(0) = z - h(1))."""
    n = xs[1]["m"].shape[0]
    if n % 2:
        pad = lambda a: np.concatenate([a, np.zeros((1, d), dtype=U)])
        xs, ys = _map(xs, pad), _map(ys, pad)
    f0, f1 = _map(xs, lambda a: a[0::2]), _map(xs, lambda a: a[1::2])
    g0, g1 = _map(ys, lambda a: a[0::2]), _map(ys, lambda a: a[1::2])
    two = lambda a: _wrap(lambda: (a * U(2)) & _m(ell))
    f2 = _zip(_map(f1, two), f0, lambda a, b: _sub(a, b, ell))
    g2 = _zip(_map(g1, two), g0, lambda a, b: _sub(a, b, ell))
    h1 = gr_dot(sim, f1, g1, ell, d)
    h2 = gr_dot(sim, f2, g2, ell, d)
    h0 = _zip(z, h1, lambda a, b: _sub(a, b, ell))
    ze = rec(sim, _map(zeta, two), "vfy.zeta", ell, d, style="challenge")
    sim.barrier()
    l0, l1, l2 = gr.quad_coeffs(ze, ell, d)
    z_out = _zip(_zip(_scale_gr(h0, l0, ell, d), _scale_gr(h1, l1, ell, d),
                      lambda a, b: _add(a, b, ell)),
                 _scale_gr(h2, l2, ell, d), lambda a, b: _add(a, b, ell))
    line = lambda p0, p1: _zip(p0, _scale_gr(_zip(p1, p0, lambda a, b: _sub(a, b, ell)), ze, ell, d),
                               lambda a, b: _add(a, b, ell))
    return line(f0, f1), line(g0, g1), z_out


def check_inner_product(sim, xs, ys, z, ell, d, alpha):
    """verify.py:244-263."""
    M = xs[1]["m"].shape[0]
    gid = sim.next_id("vfy.amul")
    out = sha_random(sim, M, ell, d)
    cross = gr.mul(xs[0]["total"], alpha[0]["total"], ell, d)
    g = sha_input(sim, _add(cross, out[0]["total"], ell), M, ell, d, f"vfy.amul.gamma.{gid}", "offline")
    mul = lambda a, b: gr.mul(a, b, ell, d)
    leg1 = _sub(_sub(g[1]["s1"], mul(xs[1]["m"], alpha[1]["s1"]), ell), mul(alpha[1]["m"], xs[1]["s1"]), ell)
    leg2 = _sub(_sub(_add(mul(xs[2]["m"], alpha[2]["m"]), g[2]["s2"], ell),
                     mul(xs[2]["m"], alpha[2]["s2"]), ell), mul(alpha[2]["m"], xs[2]["s2"]), ell)
    sim.send(1, 2, f"vfy.amul.mz.{gid}.leg1", M * d, ell)
    sim.send(2, 1, f"vfy.amul.mz.{gid}.leg2", M * d, ell, "aux")
    mz = _add(leg1, leg2, ell)
    xp = {r: dict(out[r]) for r in range(3)}
    xp[1]["m"] = mz
    xp[2]["m"] = mz
    cat = lambda a, b: np.concatenate([a, b])
    pairs_x = _zip(xp, alpha, cat)
    negz = _map(z, lambda a: _wrap(lambda: (U(0) - a) & _m(ell)))
    pairs_y = _zip(ys, negz, cat)
    delta = gr_dot(sim, pairs_x, pairs_y, ell, d)
    opened = rec(sim, delta, "vfy.delta", ell, d, style="aux")
    sim.barrier()
    return bool(np.all(opened == 0))


def lift(v, d):
    """verify.py:126-140: P0 keeps only the mask sum."""
    out = {0: {"total": gr.embed(v[0]["total"], d)}}
    for r in (1, 2):
        out[r] = {k: gr.embed(v[r][k], d) for k in _comps(r)}
    return out


def batch_verify_muls(sim, x, y, z, ell, d, R, chal):
    """verify.py:278-311 for a single multiplication batch."""
    r = rec(sim, chal["r"], "vfy.r", ell, d, style="challenge")
    sim.barrier()
    n = x[1]["m"].shape[0]
    pw = gr.powers(r, n, ell, d)
    xg = _scale_gr(lift(x, d), pw, ell, d)
    yg = lift(y, d)
    zg = _map(_scale_gr(lift(z, d), pw, ell, d),
              lambda a: _wrap(lambda: (a.sum(axis=0, dtype=U) & _m(ell)).reshape(1, d)))
    for k in range(R):
        xg, yg, zg = reduce_dimension(sim, xg, yg, zg, ell, d, chal["zetas"][k])
    return check_inner_product(sim, xg, yg, zg, ell, d, chal["alpha"])


def prepare_verification(sim, ell, d, r_max):
    """verify.py:101-119: sealed r, alpha, zeta_1..r_max per log kind."""
    ctx = {}
    for kind in ("mul.arith", "dot.arith", "mul.bool"):
        w = 1 if kind.endswith("bool") else ell
        ctx[kind] = {"r": shc_random(sim, 1, w, d), "alpha": shc_random(sim, 1, w, d),
                     "zetas": [shc_random(sim, 1, w, d) for _ in range(r_max)]}
    return ctx


# ---------------------------------------------------------------------------
# programs
# ---------------------------------------------------------------------------

@dataclass
class MulvResult:
    x: dict
    y: dict
    z: dict
    verdict: bool
    sim: Sim
    counters: dict = field(default_factory=dict)

    def rounds_by_phase(self, Phase):
        return self.sim.rounds_by_phase(Phase)


def mulv(seed: int, lanes: int, d: int, R: int, ell: int = 64, r_max: int | None = None) -> MulvResult:
    """The mulv program of tests/test_acceptance.py:124-136 (shc_random x, y;
    one Pi_mul; prepare_verification; batch_verify_muls)."""
    sim = Sim(seed, ell)
    x = shc_random(sim, lanes, ell)
    y = shc_random(sim, lanes, ell)
    gid, out, g = mul_gate(sim, x, y, lanes, ell)
    ctx = prepare_verification(sim, ell, d, max(R, 1) if r_max is None else r_max)
    sim.barrier()
    sim.phase = ONLINE
    z = mul_finish(sim, gid, out, g, x, y, lanes, ell)
    sim.barrier()
    sim.phase = POST
    verdict = batch_verify_muls(sim, x, y, z, ell, d, R, ctx["mul.arith"])
    return MulvResult(x, y, z, verdict, sim, dict(sim.counters))
