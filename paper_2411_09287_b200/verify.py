"""Postprocessing batch verification over GR(2^ell, d) on the GPU.

Drop-in for the reference `ring3pc.verify` (verify.py:1-338): the same cost
model, challenge draws, message flow, accounting classes and verdicts.  The
pipeline is Pi_tran (compress the logged triples with challenge powers
r^0, r^1, ...) -> R x Pi_rd (halve the inner-product dimension by line
interpolation; h(1), h(2) by inner products, h(0) = z - h(1), evaluation at
an opened even point) -> Pi_vdot (random multiplier alpha, fold in the
claimed result, open, test for zero).

B200 structure (SURVEY.md findings 4-5):

* The compressed vectors x'_i = r^i x_i and y'_i = y_i are never
  materialised.  Compression and the first reduction are fused: one pass
  over the base-ring log computes each party's h(1)/h(2) folds against the
  challenge-power table (r3_vfy_l1_fold, d MACs per term instead of the
  reference's d^2 schoolbook on lifted arrays), a second pass writes the
  level-1 vectors directly from two public tables A_j = r^{2j}(1-zeta),
  B_j = r^{2j+1} zeta (r3_vfy_l1_line_x / _y).  The power table and the
  public tables are computed once per session and shared by the three
  simulated parties (they are public values every party derives
  identically; the cache is keyed by the opened bytes).
* Later levels operate on dense (N_k, d) arrays: inner products as
  sum_i F_i (x) G_i (r3_gr_dotsum) and line evaluations as rows . M_zeta
  (r3_gr_matmul).
"""

from __future__ import annotations

import math
import os
import threading
from dataclasses import dataclass

import ctypes as C
import torch

from . import grvec
from ._lib import call, empty, ptr, stream, to_host
from .gates import MatmulBatchRec, MulBatchRec, dot_finish, dot_prepare, prepare_gate
from .rings import ConfigError, modulus_for_degree
from .sharing import AShare, MVal, Ring, rec, shc_random
from .transport import AUX, OFFLINE, PAYLOAD, HarnessError, Phase

CHALLENGE_KINDS = ("mul.arith", "dot.arith", "mul.bool")
DEFAULT_R_MAX = 24


# ---------------------------------------------------------------------------
# cost model (verify.py:49-87)
# ---------------------------------------------------------------------------

def online_bits(gates: int, R: int, ell: int, d: int) -> int:
    return (5 * R + 3 + math.ceil(gates / 2 ** R)) * ell * d


def offline_bits(gates: int, R: int, ell: int, d: int) -> int:
    return (R + math.ceil(gates / 2 ** R)) * ell * d


def rounds(R: int) -> int:
    return R + 2


NETWORK_PROFILES = {
    # round-trip time (ms), bandwidth (bit/s)
    "lan": (0.2, 1e9),
    "man": (12.0, 1e8),
    "wan": (80.0, 4e7),
}


def latency_estimate(n_rounds: int, bits: int, profile: str) -> float:
    """rounds * RTT + bits / bandwidth, in milliseconds."""
    rtt, bw = NETWORK_PROFILES[profile]
    return n_rounds * rtt + bits / bw * 1000.0


def pick_r(gates: int, ell: int, d: int, profile: str = "lan", r_max: int = DEFAULT_R_MAX) -> int:
    """Reduction count minimising the modelled latency (first minimum wins)."""
    if gates <= 1:
        return 0
    best_r, best = 0, None
    for R in range(min(r_max, int(math.log2(gates))) + 1):
        bits = online_bits(gates, R, ell, d) + offline_bits(gates, R, ell, d)
        cost = latency_estimate(rounds(R), bits, profile)
        if best is None or cost < best:
            best_r, best = R, cost
    return best_r


# ---------------------------------------------------------------------------
# challenges (verify.py:94-119)
# ---------------------------------------------------------------------------

@dataclass
class Challenges:
    r: MVal
    alpha: MVal
    zetas: "_SealedBlock"


def prepare_verification(party, d: int, r_max: int = DEFAULT_R_MAX) -> None:
    """Sealed extension-ring challenges for every log kind, drawn in PRE."""
    if party.phase is not Phase.PRE:
        raise ConfigError("verification challenges must be drawn in preprocessing")
    mod = modulus_for_degree(d)
    ctx = {}
    for kind in CHALLENGE_KINDS:
        gr = Ring(1 if kind.endswith("bool") else party.ell, mod)
        ch = _sealed_block(party, 2 + r_max, gr)
        ctx[kind] = Challenges(r=ch[0], alpha=ch[1], zetas=ch[2:])
    party.verify_ctx = ctx


class _SealedBlock:
    """A read-only sequence of sealed challenge shares over one block of
    keystream words; the MVal of value k is built when it is first read (a
    verification opens R + 2 of the r_max + 2 prepared values)."""

    def __init__(self, make, count: int, start: int = 0):
        self._make, self._n, self._start = make, count, start
        self._cache = {}

    def __len__(self) -> int:
        return self._n

    def __getitem__(self, k):
        if isinstance(k, slice):
            lo, hi, step = k.indices(self._n)
            if step != 1:
                raise IndexError("sealed challenge blocks slice contiguously")
            return _SealedBlock(self._make, max(0, hi - lo), self._start + lo)
        if k < 0:
            k += self._n
        if not 0 <= k < self._n:
            raise IndexError(k)
        v = self._cache.get(k)
        if v is None:
            v = self._cache[k] = self._make(self._start + k)
        return v

    def __iter__(self):
        return (self[k] for k in range(self._n))


def _sealed_block(party, count: int, gr: Ring) -> _SealedBlock:
    """`count` consecutive shc_random(party, 1, gr, seal=True) values
    (sharing.py:316-321) with one keystream draw per pairwise stream: each
    stream's offsets advance exactly as `count` single draws would (P0 "01"
    then "02" per value, m from "12"), so every share is identical."""
    role = party.role
    draw = lambda pair, dom: party.prg(pair, dom).draw_gr(count, gr.ell, gr.mod)
    if role == 0:
        s1, s2 = draw("01", "sha"), draw("02", "sha")
        tot = grvec.add(s1, s2, gr.ell)
        return _SealedBlock(lambda k: MVal(AShare(gr, 0, s1=s1[k:k + 1], s2=s2[k:k + 1], total=tot[k:k + 1]),
                                           None, sealed=True), count)
    half = "s1" if role == 1 else "s2"
    h = draw("01" if role == 1 else "02", "sha")
    m = draw("12", "sha.m")
    return _SealedBlock(lambda k: MVal(AShare(gr, role, **{half: h[k:k + 1]}), m[k:k + 1], sealed=True), count)


# ---------------------------------------------------------------------------
# share plumbing over the extension ring
# ---------------------------------------------------------------------------

def _lift(v: MVal, gr: Ring) -> MVal:
    """Base -> extension share (constant coefficient).  P0 keeps only its mask
    sums (verify.py:126-140)."""
    emb = lambda a: None if a is None else grvec.gr_embed(a, gr.mod)
    p0 = v.mask.role == 0
    mask = AShare(gr, v.mask.role, s1=None if p0 else emb(v.mask.s1),
                  s2=None if p0 else emb(v.mask.s2), total=emb(v.mask.total),
                  p0_halves=False if p0 else v.mask.p0_halves)
    return MVal(mask, emb(v.m))


def _zero_lanes(party, gr: Ring, lanes: int) -> MVal:
    return MVal(AShare.zero(gr, party.role, lanes), gr.zeros(lanes) if party.role in (1, 2) else None)


def _sum_lanes(v: MVal, gr: Ring) -> MVal:
    red = lambda a: grvec.sum_axis0(a, gr.ell, keepdims=True)
    return MVal(v.mask._map(red), None if v.m is None else red(v.m))


def _gr_dot(party, xs: MVal, ys: MVal, gr: Ring, leg2_cls: str = PAYLOAD) -> MVal:
    """(N, d) x (N, d) -> (1, d) inner product; Gamma booked as "offline"."""
    unsq = lambda v: MVal(v.mask._map(lambda a: a[:, None]),
                          None if v.m is None else v.m[:, None], v.sealed)
    x2, y2 = unsq(xs), unsq(ys)
    gate = dot_prepare(party, x2.mask, y2.mask, lanes=1, kind="vfy.dot", gamma_cls=OFFLINE)
    return dot_finish(party, gate, x2, y2, log=False, leg2_cls=leg2_cls)


def _gr_dot_folded(party, gr: Ring, n: int, fold: torch.Tensor, leg2_cls: str = PAYLOAD) -> MVal:
    """_gr_dot with the party's local fold precomputed by a fused kernel:
    P0's cross term, or the sum of P1/P2's leg products (without Gamma)."""
    gate = prepare_gate(party, gr, n, 1, None, "vfy.dot", OFFLINE, lambda: fold)
    if party.role == 0:
        return dot_finish(party, gate, None, None, log=False, leg2_cls=leg2_cls)
    g = gate.gamma.s1 if party.role == 1 else gate.gamma.s2
    leg = grvec.add(fold, g, gr.ell)
    return dot_finish(party, gate, None, None, log=False, leg2_cls=leg2_cls, leg=leg)


# ---------------------------------------------------------------------------
# public tables shared by the three simulated parties
# ---------------------------------------------------------------------------

_cache_lock = threading.Lock()


def _public(party, key, build):
    sess = party.sess
    cache = sess.public_cache
    with _cache_lock:
        if key not in cache:
            cache[key] = build()
            group = party._vgroup
            if group is not None:
                sess.public_groups.setdefault(group, []).append(key)
        return cache[key]


def _verification_group(party, name: str, run):
    """Run one log's verification; the public tables it builds (powers,
    line / level tables) are dropped as soon as all three parties have
    finished that log, so the logs of a session verify one after the other
    at the largest one's peak instead of the sum."""
    group = (name, party.next_id("_vgroup"))
    party._vgroup = group
    try:
        return run()
    finally:
        party._vgroup = None
        sess = party.sess
        with _cache_lock:
            done = sess.public_groups_done[group] = sess.public_groups_done.get(group, 0) + 1
            if done == 3:
                del sess.public_groups_done[group]
                for key in sess.public_groups.pop(group, ()):
                    sess.public_cache.pop(key, None)


def _shared_m(party, build):
    """The masked value m is held identically by P1 and P2 in an honest
    session, so anything computed from m alone (line evaluations of the m
    component) is computed once: the first of the two to arrive builds it,
    the second takes the same tensor (value semantics: nothing writes into
    it).  Sessions with an adversary, and the threads engine, compute per
    party as in the reference."""
    if party.role == 0 or not _joint_ok(party):
        return build()
    key = ("m", party.next_id("_shared_m"))
    memo = party.sess.shared_m
    if key in memo:
        return memo.pop(key)
    out = memo[key] = build()
    return out


def _opened_key(party, value: torch.Tensor):
    """Cache identity of a just-opened public value.  With eager checks (an
    adversary is configured) parties may disagree on an opening until the
    digest check aborts, so the key is the opened bytes themselves; in
    honest sessions every party opens the same value under the same rec tag,
    so the tag identifies it without a device->host read."""
    if party.sess.eager_checks:
        return to_host(value).tobytes()
    return ("rec", party._ids.get("rec", 0))


class _Quad:
    """Public per-level values derived from the opened even point ze:
    Lagrange weights for z' = z l0 + h1 (l1 - l0) + h2 l2 (h0 = z - h1
    folded in) and the line-evaluation matrices of (1 - ze) and ze."""

    def __init__(self, ze: torch.Tensor, gr: Ring, check: bool):
        # one launch (r3_gr_quad): the weights, 1 - ze and, for d >= 8, the
        # multiplication matrices of 1 - ze and ze
        self.w, self.one_m, mats = grvec.gr_quad(ze, gr.ell, gr.mod, mats=gr.d >= 8, check=check)
        self.M_one_m, self.M_ze = mats if mats is not None else (None, None)


def _quad(party, ze: torch.Tensor, gr: Ring) -> _Quad:
    key = ("quad", gr.ell, gr.d, _opened_key(party, ze))
    return _public(party, key, lambda: _Quad(ze, gr, party.sess.eager_checks))


def _recombine(party, z: MVal, h1: MVal, h2: MVal, q: _Quad, gr: Ring) -> MVal:
    """z' = (z - h1) l0 + h1 l1 + h2 l2 (verify.py:233-236) over every
    field the three views share, one launch."""
    names = [f for f in ("s1", "s2", "total")
             if all(getattr(v.mask, f) is not None for v in (z, h1, h2))]
    terms = [[getattr(v.mask, f) for f in names] for v in (z, h1, h2)]
    with_m = z.m is not None
    if with_m:
        for row, v in zip(terms, (z, h1, h2)):
            row.append(v.m)
    outs = grvec.gr_lincomb(terms, list(q.w), gr.ell, gr.mod)
    vals = dict(zip(names, outs))
    mask = AShare(gr, z.mask.role, p0_halves=z.mask.p0_halves and h1.mask.p0_halves and h2.mask.p0_halves,
                  **vals)
    return MVal(mask, outs[-1] if with_m else None)


def _reduction_round(party, gr: Ring, rows: int, h1f: torch.Tensor, h2f: torch.Tensor, z: MVal, zeta: MVal):
    """The protocol steps of one reduction (verify.py:229-236) after the
    party's local folds: h(1), h(2) as Pi_dot gates of single GR elements
    (Gamma dealt by P0, legs exchanged), the opened even point ze = 2 zeta,
    its Lagrange weights and z' = (z - h1) l0 + h1 l1 + h2 l2.  Returns
    (z', ze, quad).  Honest joint sessions run the three parties' steps in
    one rendezvous (_round_joint: the same draws, messages and values, a
    handful of launches for all parties instead of about fifteen per party);
    every other session runs them gate by gate as the reference does."""
    if _joint_ok(party):
        key = ("round", party.next_id("_joint.round"))
        z2, ze, q = party.sess.joint(key, party.role, (h1f, h2f, z, zeta),
                                     lambda slots: _round_joint(party.sess, gr, rows, slots))
        party.round_barrier()
        return z2, ze, q
    h1 = _gr_dot_folded(party, gr, rows, h1f)
    h2 = _gr_dot_folded(party, gr, rows, h2f)
    ze = _open_challenge(party, zeta.scale_pub(2), "vfy.zeta")
    q = _quad(party, ze, gr)
    return _recombine(party, z, h1, h2, q, gr), ze, q


def _round_joint(sess, gr: Ring, rows: int, slots: dict) -> dict:
    """_reduction_round for all three simulated parties at once (run by the
    last party to arrive; honest joint coop session).  Per party the PRF
    streams advance exactly as in gate-by-gate execution (gates.py:52-74 via
    prepare_gate: output-mask shares, then P0's Gamma share s1, per gate)
    and every party sends its messages with the reference's labels, classes
    and per-sender order: P0 the two Gamma shares then the r1 / r2 legs of
    the opening; P1 its two legs, then m and the r1 digest; P2 its two legs,
    then the m and r2 digests.  Every send precedes its receive, so no party
    blocks inside the rendezvous."""
    P = sess.parties
    ell, d = gr.ell, gr.d
    (f01, f02, z0, zt0), (f11, f12, z1, zt1), (f21, f22, z2, zt2) = (slots[r] for r in range(3))
    if z0.mask.s1 is not None or z0.mask.total is None:
        raise HarnessError("joint reduction round: P0's running z must hold only its mask sum")
    gids = [[p.next_id("vfy.dot") for _ in range(2)] for p in P]
    # draws per stream in gate order (sha_random's mask share, then P0's
    # Gamma share s1 on the 01 stream); pairwise streams give both holders
    # the same words, so P0's tensors stand for P1's / P2's
    d01 = P[0].prg("01", "sha").draw_gr(4, ell, gr.mod)          # om1.s1, g1.s1, om2.s1, g2.s1
    d02 = P[0].prg("02", "sha").draw_gr(2, ell, gr.mod)          # om1.s2, om2.s2
    P[1].prg("01", "sha").draw_gr(4, ell, gr.mod)
    P[2].prg("02", "sha").draw_gr(2, ell, gr.mod)
    om_s1, om_s2 = d01[0::2], d02
    # every party's local arithmetic of the round in one launch (r3_vfy_round)
    cat2 = lambda a, b: torch.cat([a, b]) if a.is_contiguous() and b.is_contiguous() else \
        torch.cat([a.contiguous(), b.contiguous()])
    F0, F1, F2 = cat2(f01, f02), cat2(f11, f12), cat2(f21, f22)
    blk = empty((14, d))
    call("r3_vfy_round", d, ptr(F0), ptr(F1), ptr(F2), ptr(d01.contiguous()), ptr(d02.contiguous()),
         ptr(zt0.mask.s1.contiguous()), ptr(zt0.mask.s2.contiguous()), ptr(zt1.m.contiguous()), ptr(blk),
         gr.mask, stream())
    om_tot, g_s2, leg1, leg2, m = blk[0:2], blk[2:4], blk[4:6], blk[6:8], blk[8:10]
    S1, S2, M, ze = blk[10:11], blk[11:12], blk[12:13], blk[13:14]
    for g in range(2):
        gid = gids[0][g]
        P[0].send(2, f"sha.vfy.dot.gamma.{gid}", g_s2[g:g + 1], gr, cls=OFFLINE, site="vfy.dot.gamma", gate=gid)
        P[2].recv(0, f"sha.vfy.dot.gamma.{gids[2][g]}", gr, 1)
        l1, l2 = f"vfy.dot.mz.{gids[1][g]}", f"vfy.dot.mz.{gids[2][g]}"
        P[1].send(2, f"{l1}.leg1", leg1[g:g + 1], gr, cls=PAYLOAD, site="vfy.dot.mz", gate=gids[1][g])
        P[2].send(1, f"{l2}.leg2", leg2[g:g + 1], gr, cls=PAYLOAD, site="vfy.dot.mz", gate=gids[2][g])
        P[1].recv(2, f"{l1}.leg2", gr, 1)
        P[2].recv(1, f"{l2}.leg1", gr, 1)
    # open ze = 2 zeta (sharing.rec, style "challenge"): P0's halves stand
    # for P1's s1 / P2's s2, P1's m for P2's
    tags = [f"vfy.zeta#{p.next_id('rec')}" for p in P]
    L = lambda r, leg: f"rec.{tags[r]}.{leg}"
    P[0].send(2, L(0, "r1"), S1, gr, cls=AUX)
    P[0].send(1, L(0, "r2"), S2, gr, cls=AUX)
    P[1].send(0, L(1, "m"), M, gr, cls=PAYLOAD)
    P[1].send_digest(2, L(1, "r1"), S1, gr)
    P[2].send_digest(0, L(2, "m"), M, gr)
    P[2].send_digest(1, L(2, "r2"), S2, gr)
    m0 = P[0].recv(1, L(0, "m"), gr, 1)
    P[0].check_digest(2, L(0, "m"), m0, gr, f"rec {tags[0]} m")
    s2_1 = P[1].recv(0, L(1, "r2"), gr, 1)
    P[1].check_digest(2, L(1, "r2"), s2_1, gr, f"rec {tags[1]} r2")
    s1_2 = P[2].recv(0, L(2, "r1"), gr, 1)
    P[2].check_digest(1, L(2, "r1"), s1_2, gr, f"rec {tags[2]} r1")
    q = _quad(P[0], ze, gr)
    # z' for every party's fields in one launch: P0 total, P1 s1, P2 s2, m
    w = list(q.w)
    terms = [[z0.mask.total, z1.mask.s1, z2.mask.s2, z1.m],
             [om_tot[0:1], om_s1[0:1], om_s2[0:1], m[0:1]],
             [om_tot[1:2], om_s1[1:2], om_s2[1:2], m[1:2]]]
    o_tot, o_s1, o_s2, o_m = grvec.gr_lincomb(terms, w, ell, gr.mod)
    return {0: (MVal(AShare(gr, 0, total=o_tot, p0_halves=False), None), ze, q),
            1: (MVal(AShare(gr, 1, s1=o_s1, p0_halves=z1.mask.p0_halves), o_m), ze, q),
            2: (MVal(AShare(gr, 2, s2=o_s2, p0_halves=z2.mask.p0_halves), o_m), ze, q)}


def _powers(party, r: torch.Tensor, n: int, gr: Ring) -> torch.Tensor:
    key = ("pow", gr.ell, gr.d, _opened_key(party, r), n)
    return _public(party, key, lambda: grvec.gr_powers(r, n, gr.ell, gr.mod))


def _powers4(party, r: torch.Tensor, n4: int, gr: Ring):
    """(r^(4j) for j < n4, r^0..r^3): the table of every fourth power and the
    four in-block offsets (pw[4j + a] = pw4[j] r^a)."""
    key = ("pow4", gr.ell, gr.d, _opened_key(party, r), n4)

    def build():
        rpow = grvec.gr_powers(r, 5, gr.ell, gr.mod)
        return grvec.gr_powers(rpow[4:5], n4, gr.ell, gr.mod), rpow[:4].contiguous()
    return _public(party, key, build)


def _line_tables(party, r, pw: torch.Tensor, dot_n: int, ze: torch.Tensor, gr: Ring):
    """Public level-1 tables A = pw (1 - ze), B = pw ze.  For multiplication
    logs (dot_n == 1) only even powers feed A and odd powers feed B."""
    key = ("ab", gr.ell, gr.d, id(pw), pw.shape[0], dot_n, _opened_key(party, ze))

    def build():
        one = grvec.gr_const(1, gr.mod, gr.ell)
        one_m = grvec.sub(one, ze, gr.ell)
        M_a = grvec.gr_mulmat(one_m, gr.mod) if gr.d >= 8 else None
        M_b = grvec.gr_mulmat(ze, gr.mod) if gr.d >= 8 else None
        ev, od = (pw[0::2], pw[1::2]) if dot_n == 1 else (pw, pw)
        if gr.d >= 8:
            A = grvec.rows_times(ev, M_a, ev.shape[0], gr.ell)
            B = grvec.rows_times(od, M_b, od.shape[0], gr.ell) if od.shape[0] else empty((0, gr.d))
        else:
            A = grvec.gr_mul(ev.contiguous(), one_m, gr.ell, gr.mod)
            B = grvec.gr_mul(od.contiguous(), ze, gr.ell, gr.mod) if od.shape[0] else empty((0, gr.d))
        return A, B, one_m
    return _public(party, key, build)


# ---------------------------------------------------------------------------
# compressed (never materialised) base-ring logs
# ---------------------------------------------------------------------------

@dataclass
class _Compressed:
    """x'_i = pw[i // n] * x_i, y'_i = y_i: base components of a log laid out
    (n, L) (element i at (i % n, i // n)); n = 1 for multiplication logs."""

    x: dict
    y: dict
    n: int
    N: int
    ks: int
    ls: int


def _components(v: MVal, role: int) -> dict:
    """The components a party carries through verification after _lift."""
    if role == 0:
        return {"total": v.mask.total}
    name = "s1" if role == 1 else "s2"
    return {name: getattr(v.mask, name), "m": v.m}


def _compressed_from_log(xs: MVal, ys: MVal, role: int, n: int) -> _Compressed:
    xc, yc = _components(xs, role), _components(ys, role)
    a = next(iter(xc.values()))
    if n == 1:
        a = a.reshape(-1)
        xc = {k: t.reshape(-1) for k, t in xc.items()}
        yc = {k: t.reshape(-1) for k, t in yc.items()}
        strides = {t.stride(0) for t in list(xc.values()) + list(yc.values())}
        if strides != {1}:
            xc = {k: t.contiguous() for k, t in xc.items()}
            yc = {k: t.contiguous() for k, t in yc.items()}
        return _Compressed(xc, yc, 1, a.shape[0], 0, 1)
    # dot log: (n, L) arrays; all components share one stride pattern
    xc = {k: t.contiguous() for k, t in xc.items()}
    yc = {k: t.contiguous() for k, t in yc.items()}
    L = a.shape[1]
    return _Compressed(xc, yc, n, n * L, L, 1)


def _ptrs(ts):
    arr = (C.c_void_p * len(ts))(*[ptr(t) for t in ts])
    return arr


def _role_terms(role: int):
    """Leg products of _gr_dot per role as (coef, x-comp, y-comp):
    P0 cross; P1 -(m_x s_y) - (s_x m_y); P2 m_x m_y - m_x s_y - s_x m_y
    (gates.py:100-106 with the lifted x on the left)."""
    if role == 0:
        return [(1, "total", "total")]
    s = "s1" if role == 1 else "s2"
    if role == 1:
        return [(-1, "m", s), (-1, s, "m")]
    return [(1, "m", "m"), (-1, "m", s), (-1, s, "m")]


def _l1_folds(party, comp: _Compressed, pw: torch.Tensor, gr: Ring):
    terms = _role_terms(party.role)
    d = gr.d
    coef = (C.c_int64 * len(terms))(*[t[0] for t in terms])
    xs = _ptrs([comp.x[t[1]] for t in terms])
    ys = _ptrs([comp.y[t[2]] for t in terms])
    h1 = empty((1, d))
    h2 = empty((1, d))
    call("r3_vfy_l1_fold", len(terms), coef, xs, ys, comp.N, comp.n, comp.ks, comp.ls, ptr(pw),
         d, ptr(h1), ptr(h2), gr.mask, stream())
    return h1, h2


def _base_fold(party, comp: _Compressed, zcomps: list, z_stride: int, pw: torch.Tensor, gr: Ring):
    """r3_vfy_base_fold: (zsum (nz, 1, d), acc (16, d), h1 fold, h2 fold).
    Honest coop sessions run the three parties' folds in one launch that
    streams the public power table once (r3_vfy_base_fold_multi)."""
    mine = {"terms": _role_terms(party.role), "x": comp.x, "y": comp.y, "z": zcomps}
    d = gr.d

    def folds(slots):
        roles = sorted(slots)
        np_ = len(roles)
        nterms = (C.c_int * np_)(*[len(slots[r]["terms"]) for r in roles])
        nz = (C.c_int * np_)(*[len(slots[r]["z"]) for r in roles])
        coef = (C.c_int64 * (3 * np_))()
        xs, ys, zp = (C.c_void_p * (3 * np_))(), (C.c_void_p * (3 * np_))(), (C.c_void_p * (2 * np_))()
        out = {}
        for q, r in enumerate(roles):
            sl = slots[r]
            for t, (cf, xk, yk) in enumerate(sl["terms"]):
                coef[3 * q + t], xs[3 * q + t], ys[3 * q + t] = cf, ptr(sl["x"][xk]), ptr(sl["y"][yk])
            for c, zt in enumerate(sl["z"]):
                zp[2 * q + c] = ptr(zt)
            out[r] = (empty((len(sl["z"]), 1, d)), empty((16, d)), empty((1, d)), empty((1, d)))
        zs = (C.c_int64 * np_)(*([z_stride] * np_))
        arrs = [(C.c_void_p * np_)(*[ptr(out[r][i]) for r in roles]) for i in range(4)]
        call("r3_vfy_base_fold_multi", np_, C.addressof(nterms), C.addressof(coef), C.addressof(xs),
             C.addressof(ys), C.addressof(nz), C.addressof(zp), C.addressof(zs), comp.N, ptr(pw), d,
             C.addressof(arrs[1]), C.addressof(arrs[2]), C.addressof(arrs[3]), C.addressof(arrs[0]),
             gr.mask, stream())
        return out

    if _joint_ok(party):
        return party.sess.joint(("bfold", party.next_id("_joint.bfold")), party.role, mine, folds)
    return folds({party.role: mine})[party.role]


def _base_fold_q4(party, comp: _Compressed, zcomps: list, z_stride: int, q4, gr: Ring):
    """_base_fold against the r^(4j) table (r3_vfy_base_fold_q4): the raw
    accumulators sum_j s^{ab}_j r^(4j) and sum_j z[4j+a] r^(4j) are taken
    times r^a here, then the level-1 folds follow (r3_vfy_base_fold_finish)."""
    pw4, rpow = q4
    mine = {"terms": _role_terms(party.role), "x": comp.x, "y": comp.y, "z": zcomps}
    d = gr.d
    r_acc = rpow.repeat_interleave(4, dim=0)          # row a*4 + b -> r^a

    def folds(slots):
        roles = sorted(slots)
        np_ = len(roles)
        nterms = (C.c_int * np_)(*[len(slots[r]["terms"]) for r in roles])
        nz = (C.c_int * np_)(*[len(slots[r]["z"]) for r in roles])
        coef = (C.c_int64 * (3 * np_))()
        xs, ys, zp = (C.c_void_p * (3 * np_))(), (C.c_void_p * (3 * np_))(), (C.c_void_p * (2 * np_))()
        raw = {}
        for q, r in enumerate(roles):
            sl = slots[r]
            for t, (cf, xk, yk) in enumerate(sl["terms"]):
                coef[3 * q + t], xs[3 * q + t], ys[3 * q + t] = cf, ptr(sl["x"][xk]), ptr(sl["y"][yk])
            for c, zt in enumerate(sl["z"]):
                zp[2 * q + c] = ptr(zt)
            raw[r] = (empty((16, d)), empty((max(1, len(sl["z"])) * 4, d)))
        zs = (C.c_int64 * np_)(*([z_stride] * np_))
        arrs = [(C.c_void_p * np_)(*[ptr(raw[r][i]) for r in roles]) for i in range(2)]
        call("r3_vfy_base_fold_q4", np_, C.addressof(nterms), C.addressof(coef), C.addressof(xs),
             C.addressof(ys), C.addressof(nz), C.addressof(zp), C.addressof(zs), comp.N, ptr(pw4), d,
             C.addressof(arrs[0]), C.addressof(arrs[1]), stream())
        out = {}
        for r in roles:
            acc_raw, z_raw = raw[r]
            nzr = len(slots[r]["z"])
            acc = grvec.gr_mul(acc_raw, r_acc, gr.ell, gr.mod)
            zsum = empty((nzr, 1, d))
            if nzr:
                zc = grvec.gr_mul(z_raw[:4 * nzr], rpow.repeat(nzr, 1), gr.ell, gr.mod)
                for c in range(nzr):
                    zsum[c] = grvec.sum_axis0(zc[4 * c:4 * c + 4], gr.ell, keepdims=True)
            h1, h2 = empty((1, d)), empty((1, d))
            call("r3_vfy_base_fold_finish", d, nzr, ptr(acc), ptr(h1), ptr(h2), ptr(zsum), gr.mask, stream())
            out[r] = (zsum, acc, h1, h2)
        return out

    if _joint_ok(party):
        return party.sess.joint(("bfold4", party.next_id("_joint.bfold4")), party.role, mine, folds)
    return folds({party.role: mine})[party.role]


def _powsum(comps: list, stride: int, lanes: int, pw: torch.Tensor, gr: Ring) -> torch.Tensor:
    out = empty((len(comps), 1, gr.d))
    call("r3_vfy_powsum", len(comps), _ptrs(comps), stride, lanes, ptr(pw), gr.d, ptr(out),
         gr.mask, stream())
    return out


def _mval_from(comps: dict, gr: Ring, role: int) -> MVal:
    if role == 0:
        return MVal(AShare(gr, 0, total=comps["total"], p0_halves=False), None)
    s = "s1" if role == 1 else "s2"
    return MVal(AShare(gr, role, **{s: comps[s]}), comps["m"])


def _open_challenge(party, v: MVal, tag: str) -> torch.Tensor:
    out = rec(party, v, tag, style="challenge")
    party.round_barrier()
    return out


def _compress_reduce_first(party, comp: _Compressed, zs: MVal, z_lanes: int, z_stride: int,
                           gr: Ring, chal: Challenges, R: int):
    """Pi_tran fused with the first Pi_rd (verify.py:168-179 + 215-241 at
    k = 0); returns dense level-1 (xs, ys, z)."""
    r = _open_challenge(party, chal.r, "vfy.r")
    n_pw = (comp.N + comp.n - 1) // comp.n
    zc = _components(zs, party.role)
    zc = {k: t.reshape(-1) if t.dim() == 1 else t for k, t in zc.items()}
    names = list(zc)
    base_acc = q4 = pw = None
    base_ok = (R >= 2 and gr.d >= 8 and comp.n == 1 and comp.ls == 1 and z_lanes == comp.N
               and len(names) <= 2)
    B = _base_block(comp, R, gr) if base_ok else 0
    if B:
        # log2 B reductions from one pass over r^(Bj): the dense tail starts
        # at level log2 B (N / B rows)
        return _reduce_from_base(party, comp, [zc[k] for k in names], names, z_stride, r, B, gr, chal)
    if base_ok and gr.d == 64:
        # one pass over the table r^(4j) on the tensor cores: z power sum,
        # level-2 accumulators and the level-1 folds derived from them; the
        # full power table is never built (every later table is r^(4j)
        # times a constant)
        q4 = _powers4(party, r, (comp.N + 3) // 4, gr)
        zsum, base_acc, h1f, h2f = _base_fold_q4(party, comp, [zc[k] for k in names], z_stride, q4, gr)
    elif base_ok:
        # CUDA-core degrees: the same pass over the full power table
        pw = _powers(party, r, n_pw, gr)
        zsum, base_acc, h1f, h2f = _base_fold(party, comp, [zc[k] for k in names], z_stride, pw, gr)
    else:
        pw = _powers(party, r, n_pw, gr)
        zsum = _powsum([zc[k] for k in names], z_stride, z_lanes, pw, gr)
    z = _mval_from({k: zsum[i] for i, k in enumerate(names)}, gr, party.role)
    if R == 0:
        return _materialise(comp, pw, gr, party.role), z, 0
    if _lanes16_ok(comp, R, gr):
        return _reduce_lanes16(party, comp, pw, z, gr, chal)
    if base_acc is None:
        h1f, h2f = _l1_folds(party, comp, pw, gr)
    z_out, ze, _ = _reduction_round(party, gr, (comp.N + 1) // 2, h1f, h2f, z, chal.zetas[0])
    if R >= 2 and gr.d >= 8:
        return (*_reduce_second_from_base(party, comp, pw, ze, z_out, gr, chal, base_acc, q4), 2)
    A, B, one_m = _line_tables(party, r, pw, comp.n, ze, gr)
    tq = 2 if comp.n == 1 else comp.n
    half = (comp.N + 1) // 2
    xo = {k: empty((half, gr.d)) for k in comp.x}
    yo = {k: empty((half, gr.d)) for k in comp.y}
    xk, yk = list(comp.x), list(comp.y)
    call("r3_vfy_l1_line_x", len(xk), _ptrs([comp.x[k] for k in xk]), comp.N, comp.n, comp.ks,
         comp.ls, ptr(A), ptr(B), tq, gr.d, _ptrs([xo[k] for k in xk]), gr.mask, stream())
    call("r3_vfy_l1_line_y", len(yk), _ptrs([comp.y[k] for k in yk]), comp.N, comp.n, comp.ks,
         comp.ls, ptr(one_m), ptr(ze), gr.d, _ptrs([yo[k] for k in yk]), gr.mask, stream())
    xs1 = _mval_from(xo, gr, party.role)
    ys1 = _mval_from(yo, gr, party.role)
    return (xs1, ys1), z_out, 1


_LANES16_OFF = os.environ.get("R3_LANES16", "1") == "0"      # diagnostics: dot logs on the two-level form


def _lanes16_ok(comp: _Compressed, R: int, gr: Ring) -> bool:
    """Dot log (n, L) with n % 16 == 0 at d = 16 and at least four reductions."""
    return (not _LANES16_OFF and gr.d == 16 and R >= 4 and comp.n >= 16 and comp.n % 16 == 0
            and comp.ls == 1 and comp.ks * comp.n == comp.N)


def _lane_kappa(party, ws: list, gr: Ring) -> torch.Tensor:
    """kappa_a = prod_{l < 4} ws[l][bit l of a], a < 16: the line weight of
    base element 16j + a in its level-4 row."""
    key = ("lk16", gr.ell, gr.d, tuple(_opened_key(party, w[1]) for w in ws))

    def build():
        kappa = None
        for lvl, w in enumerate(ws):
            f = torch.cat([w[(a >> lvl) & 1] for a in range(16)])
            kappa = f if kappa is None else grvec.gr_mul(kappa, f, gr.ell, gr.mod)
        return kappa.contiguous()
    return _public(party, key, build)


def _reduce_lanes16(party, comp: _Compressed, pw: torch.Tensor, z: MVal, gr: Ring, chal: Challenges):
    """The first four Pi_rd of a dot log whose lanes hold a multiple of 16
    elements (verify.py:215-241 at k < 4; the edaBits inner products of
    length ell): blocks of 16 consecutive elements never straddle a lane and
    share its power r^(P+l), so every fold of those levels is a public-weight
    combination of 256 per-lane scalar sums times pw[l] (r3_vfy_lane16_fold,
    weights verify._block_fold_weights), and the level-4 rows come straight
    from the base shares (r3_vfy_lane16_line): the dense tail starts at N/16
    rows.  Returns ((xs, ys), z, 4)."""
    role, d = party.role, gr.d
    terms = _role_terms(role)
    coef = (C.c_int64 * len(terms))(*[t[0] for t in terms])
    L = comp.N // comp.n
    acc = empty((256, d))
    call("r3_vfy_lane16_fold", len(terms), coef, _ptrs([comp.x[t[1]] for t in terms]),
         _ptrs([comp.y[t[2]] for t in terms]), L, comp.n, ptr(pw), d, ptr(acc), stream())
    ws = []
    n = comp.N
    for k in range(4):
        W1, W2 = _block_fold_weights(party, k, ws, 16, gr)
        fold = lambda W: _dotsum_terms([([(1, acc, 256)], [(1, W, 256)])], 256, gr)
        rows = (n + 1) // 2
        z, ze, q = _reduction_round(party, gr, rows, fold(W1), fold(W2), z, chal.zetas[k])
        ws.append((q.one_m, ze))
        n = rows
    kappa = _lane_kappa(party, ws, gr)
    rows4 = comp.N // 16
    out = {}
    for side, src, pow_side in (("x", comp.x, 1), ("y", comp.y, 0)):
        keys = list(src)
        dst = {k: empty((rows4, d)) for k in keys}
        call("r3_vfy_lane16_line", pow_side, len(keys), _ptrs([src[k] for k in keys]), L, comp.n,
             ptr(pw) if pow_side else None, ptr(kappa), gr.mod.lowterms_mask, d, _ptrs([dst[k] for k in keys]),
             gr.mask, stream())
        out[side] = _mval_from(dst, gr, role)
    return (out["x"], out["y"]), z, 4


def _l2_weights(party, ze1: torch.Tensor, gr: Ring):
    """Public weights of the second reduction's 16 accumulators (vfy2.cu):
    W[a][b] = w_{a&1} w_{b&1} with w = (1 - ze_1, ze_1); h(1) keeps the odd
    half (a, b >= 2), h(2) weighs by alpha_a alpha_b, alpha = (-1,-1,2,2)."""
    def build():
        one = grvec.gr_const(1, gr.mod, gr.ell)
        w = (grvec.sub(one, ze1, gr.ell), ze1)
        prod = {(p, q): grvec.gr_mul(w[p], w[q], gr.ell, gr.mod) for p in (0, 1) for q in (0, 1)}
        alpha = (-1, -1, 2, 2)
        W1, W2 = [], []
        for a in range(4):
            for b in range(4):
                base = prod[(a & 1, b & 1)]
                W1.append(base if (a >= 2 and b >= 2) else grvec.zeros((1, gr.d)))
                W2.append(grvec.ew(grvec.MUL, base, alpha[a] * alpha[b], gr.mask))
        return torch.cat(W1), torch.cat(W2), w
    return _public(party, ("l2w", gr.ell, gr.d, _opened_key(party, ze1)), build)


def _reduce_second_from_base(party, comp: _Compressed, pw: torch.Tensor, ze1: torch.Tensor,
                             z1: MVal, gr: Ring, chal: Challenges, acc: torch.Tensor | None = None,
                             q4=None):
    """The second Pi_rd (verify.py:215-241 at k = 1) computed from the base
    log: 16 scalar-weighted power sums per party (r3_vfy_l2_fold) replace the
    level-1 vectors and their d^2 inner products; the level-2 vectors for the
    dense tail are written straight from the base shares (r3_vfy_line_b)."""
    role = party.role
    if acc is None:
        terms = _role_terms(role)
        coef = (C.c_int64 * len(terms))(*[t[0] for t in terms])
        acc = empty((16, gr.d))
        call("r3_vfy_l2_fold", len(terms), coef, _ptrs([comp.x[t[1]] for t in terms]),
             _ptrs([comp.y[t[2]] for t in terms]), comp.N, comp.n, comp.ks, comp.ls, ptr(pw), gr.d,
             ptr(acc), stream())
    W1, W2, w1 = _l2_weights(party, ze1, gr)
    fold = lambda W: _dotsum_terms([([(1, acc, 16)], [(1, W, 16)])], 16, gr)
    n1 = (comp.N + 1) // 2
    rows = (n1 + 1) // 2
    z2, ze2, _ = _reduction_round(party, gr, rows, fold(W1), fold(W2), z1, chal.zetas[1])
    if q4 is not None:
        tabs, kappa, tq, stride = _l2_tables_q4(party, q4, w1, ze2, gr)
    else:
        tabs, kappa, tq, stride = _l2_tables(party, pw, comp.n, w1, ze2, gr)
    geo = (comp.N, comp.n, comp.ks, comp.ls)

    def level2_vectors(slots):
        """One r3_vfy_line_b / _const launch over the components of every
        party in `slots` (the public tables are streamed once for all)."""
        nb = (comp.N + 3) // 4
        out = {}
        for side, fn, arg in (("x", "r3_vfy_line_b", None), ("y", "r3_vfy_line_b_const", None)):
            # m is the same public value at P1 and P2 (honest joint session):
            # one output serves both
            srcs = [(r, k, t) for r, sl in sorted(slots.items()) for k, t in sl[side].items()
                    if not (r == 2 and k == "m" and 1 in slots and "m" in slots[1][side])]
            dst = [empty((nb, gr.d)) for _ in srcs]
            for c0 in range(0, len(srcs), 8):
                part, pdst = srcs[c0:c0 + 8], dst[c0:c0 + 8]
                if side == "x":
                    call(fn, 4, len(part), _ptrs([t for _, _, t in part]), *geo, ptr(tabs), stride, tq,
                         gr.d, _ptrs(pdst), gr.mask, stream())
                else:
                    call(fn, 4, len(part), _ptrs([t for _, _, t in part]), *geo, ptr(kappa), gr.d,
                         _ptrs(pdst), gr.mask, stream())
            for (r, k, _), o in zip(srcs, dst):
                out.setdefault(r, {"x": {}, "y": {}})[side][k] = o
            if 2 in slots and "m" in slots[2][side] and "m" not in out.get(2, {}).get(side, {}):
                out.setdefault(2, {"x": {}, "y": {}})[side]["m"] = out[1][side]["m"]
        return out

    mine = {"x": comp.x, "y": comp.y}
    if _joint_ok(party):
        res = party.sess.joint(("l2vec", party.next_id("_joint.l2vec")), role, mine, level2_vectors)
    else:
        res = level2_vectors({role: mine})[role]
    return (_mval_from(res["x"], gr, role), _mval_from(res["y"], gr, role)), z2


# diagnostics: R3_BASE_BLOCK=0 / 8 caps the base reduction's block size
_BASE_BLOCK_CAP = int(os.environ.get("R3_BASE_BLOCK", "16"))


def _base_block(comp: _Compressed, R: int, gr: Ring) -> int:
    """Block size of the multi-level base reduction of a d = 64 / 16
    multiplication log: 16 (four reductions from the base log, dense tail
    from N/16 rows) or 8 (three, N/8), each on the tensor cores once the log
    has >= 4096 blocks; 0 = the two-level form."""
    if gr.d not in (16, 64):
        return 0
    cap = _BASE_BLOCK_CAP
    if cap < 16 and R >= 3 and comp.N >= 8 * 4096:
        return 8 if cap >= 8 else 0
    if R >= 4 and comp.N >= 16 * 4096:
        return 16
    if R >= 3 and comp.N >= 8 * 4096:
        return 8
    return 0


def _powers_b(party, r: torch.Tensor, nb: int, B: int, gr: Ring):
    """(r^(Bj) for j < nb, r^0..r^(B-1)): every B-th power and the in-block
    offsets (pw[Bj + a] = pwB[j] r^a)."""
    key = ("powb", B, gr.ell, gr.d, _opened_key(party, r), nb)

    def build():
        rpow = grvec.gr_powers(r, B + 1, gr.ell, gr.mod)
        return grvec.gr_powers(rpow[B:B + 1], nb, gr.ell, gr.mod), rpow[:B].contiguous()
    return _public(party, key, build)


def _base_fold_b(party, comp: _Compressed, zcomps: list, z_stride: int, qb, B: int, gr: Ring):
    """(zsum (nz, 1, d), acc (B^2, d)) with acc[a*B+b] = sum_j s^{ab}_j r^(Bj+a)
    and zsum_c = sum_i z_c[i] r^i, from ONE pass over the r^(Bj) table on the
    tensor cores (r3_vfy_base_fold_q8 / _q16; the raw sums over r^(Bj) are
    taken times r^a here).  Honest joint sessions fold all three parties in
    one launch (the adjacent items of a K chunk share its table rows in L2)."""
    pwb, rpow = qb
    mine = {"terms": _role_terms(party.role), "x": comp.x, "y": comp.y, "z": zcomps}
    d = gr.d
    r_acc = rpow.repeat_interleave(B, dim=0)          # row a*B + b -> r^a

    def folds(slots):
        roles = sorted(slots)
        np_ = len(roles)
        nterms = (C.c_int * np_)(*[len(slots[r]["terms"]) for r in roles])
        nz = (C.c_int * np_)(*[len(slots[r]["z"]) for r in roles])
        coef = (C.c_int64 * (3 * np_))()
        xs, ys, zp = (C.c_void_p * (3 * np_))(), (C.c_void_p * (3 * np_))(), (C.c_void_p * (2 * np_))()
        raw = {}
        for q, r in enumerate(roles):
            sl = slots[r]
            for t, (cf, xk, yk) in enumerate(sl["terms"]):
                coef[3 * q + t], xs[3 * q + t], ys[3 * q + t] = cf, ptr(sl["x"][xk]), ptr(sl["y"][yk])
            for c, zt in enumerate(sl["z"]):
                zp[2 * q + c] = ptr(zt)
            raw[r] = (empty((B * B, d)), empty((max(1, len(sl["z"])) * B, d)))
        zs = (C.c_int64 * np_)(*([z_stride] * np_))
        arrs = [(C.c_void_p * np_)(*[ptr(raw[r][i]) for r in roles]) for i in range(2)]
        call(f"r3_vfy_base_fold_q{B}", np_, C.addressof(nterms), C.addressof(coef), C.addressof(xs),
             C.addressof(ys), C.addressof(nz), C.addressof(zp), C.addressof(zs), comp.N, ptr(pwb), d,
             C.addressof(arrs[0]), C.addressof(arrs[1]), stream())
        out = {}
        for r in roles:
            acc_raw, z_raw = raw[r]
            nzr = len(slots[r]["z"])
            acc = grvec.gr_mul(acc_raw, r_acc, gr.ell, gr.mod)
            zsum = empty((nzr, 1, d))
            if nzr:
                zc = grvec.gr_mul(z_raw[:B * nzr], rpow.repeat(nzr, 1), gr.ell, gr.mod)
                for c in range(nzr):
                    zsum[c] = grvec.sum_axis0(zc[B * c:B * c + B], gr.ell, keepdims=True)
            out[r] = (zsum, acc)
        return out

    if _joint_ok(party):
        return party.sess.joint(("bfoldb", party.next_id("_joint.bfoldb")), party.role, mine, folds)
    return folds({party.role: mine})[party.role]


def _block_fold_weights(party, k: int, ws: list, B: int, gr: Ring):
    """Public weights (W1, W2), each (B^2, d), of level k's folds
    (k < log2 B) over the B^2 block accumulators: h = sum_q acc[q] (x) W[q]
    (verify.py:229-231 with the level-k vectors expanded into the base blocks
    of B).  A level-k row spans 2^k base elements a with line weight V_a =
    prod_{l<k} ws[l][bit l of a]; the pair (f0, f1) of rows spans 2^(k+1),
    bit k of a tells f0 from f1.  W1 keeps a, b both in f1; W2 weighs
    alpha_a alpha_b (alpha = -1 on f0, 2 on f1: f2 = 2 f1 - f0)."""
    key = ("bwb", B, gr.ell, gr.d, k, tuple(_opened_key(party, w[1]) for w in ws))

    def build():
        nv = 1 << k
        if k == 0:
            vals = grvec.gr_const(1, gr.mod, gr.ell)
        else:
            vals = None
            for lvl in range(k):      # V[u] for u < 2^k: bit l of u picks ws[l][.]
                w = torch.cat([ws[lvl][0], ws[lvl][1]])
                if vals is None:
                    vals = w
                else:
                    n = vals.shape[0]
                    vals = grvec.gr_mul(vals.repeat(2, 1), w.repeat_interleave(n, dim=0), gr.ell, gr.mod)
        prod = grvec.gr_mul(vals.repeat_interleave(nv, dim=0), vals.repeat(nv, 1), gr.ell, gr.mod)  # [u*nv + v]
        idx, c1, c2 = _block_fold_index(k, B, prod.device)
        rows = prod[idx]
        m = _lib_i64(gr.mask)
        W1 = (rows * c1) & m
        W2 = (rows * c2) & m
        return W1.contiguous(), W2.contiguous()
    return _public(party, key, build)


_BF_INDEX: dict = {}


def _block_fold_index(k: int, B: int, dev):
    """Device constants of _block_fold_weights for level k and block size B:
    the product row of each accumulator and its integer coefficients in W1 /
    W2.  Built once per process and device (a host list -> device copy
    synchronises the stream, which the protocol driver must not do per
    session)."""
    key = (k, B, dev)
    hit = _BF_INDEX.get(key)
    if hit is None:
        nv = 1 << k
        idx, c1, c2 = [], [], []
        alpha = (-1, 2)
        for a in range(B):
            for b in range(B):
                same = (a >> (k + 1)) == (b >> (k + 1))
                ba, bb = (a >> k) & 1, (b >> k) & 1
                idx.append((a & (nv - 1)) * nv + (b & (nv - 1)))
                c1.append(1 if same and ba and bb else 0)
                c2.append(alpha[ba] * alpha[bb] if same else 0)
        hit = _BF_INDEX[key] = (torch.tensor(idx, device=dev), torch.tensor(c1, device=dev)[:, None],
                                torch.tensor(c2, device=dev)[:, None])
    return hit


def _lib_i64(v: int) -> int:
    v &= (1 << 64) - 1
    return v - (1 << 64) if v >> 63 else v


_K16_OFF = os.environ.get("R3_K16_TC", "1") == "0"     # diagnostics: y-side level-4 rows on the CUDA cores
_MUL16_OFF = os.environ.get("R3_MUL16", "1") == "0"    # diagnostics: d = 16 level-4 rows through the B tables
_TABLE_Q = int(os.environ.get("R3_TABLE_Q", "4"))      # tables per pass over r^(Bj) (4 or 2)


def _reduce_from_base(party, comp: _Compressed, zlist: list, znames: list, z_stride: int,
                      r: torch.Tensor, B: int, gr: Ring, chal: Challenges):
    """Pi_tran and the first L = log2 B Pi_rd (verify.py:168-179 + 215-241
    at k < L) from the base log: the B^2 accumulators of blocks of B
    (r3_vfy_base_fold_q8 / _q16) give every level's h(1)/h(2) folds through
    public weights, and the level-L vectors for the dense tail are written
    straight from the base shares with the public tables V_a[j] = r^(Bj)
    (r^a kappa_a) (r3_gr_matmul_q_tc, then r3_vfy_line_b with blocks of B).
    Returns ((xs, ys), z, L)."""
    role = party.role
    levels = B.bit_length() - 1
    nb = (comp.N + B - 1) // B
    qb = _powers_b(party, r, nb, B, gr)
    zsum, acc = _base_fold_b(party, comp, zlist, z_stride, qb, B, gr)
    z = _mval_from({k: zsum[i] for i, k in enumerate(znames)}, gr, role)
    ws = []
    n = comp.N
    for k in range(levels):
        W1, W2 = _block_fold_weights(party, k, ws, B, gr)
        fold = lambda W: _dotsum_terms([([(1, acc, B * B)], [(1, W, B * B)])], B * B, gr)
        rows = (n + 1) // 2
        z, ze, q = _reduction_round(party, gr, rows, fold(W1), fold(W2), z, chal.zetas[k])
        ws.append((q.one_m, ze))
        n = rows
    # d = 16, blocks of sixteen: the level-4 rows straight from the base
    # shares and r^(16j) (r3_vfy_mul16_line), no tables
    rows16 = B == 16 and gr.d == 16 and not _MUL16_OFF and qb[0].is_contiguous()
    if rows16:
        _, kappa, rk = _base_tables(party, qb, ws, B, gr, tables=False)
    else:
        tabs, kappa = _base_tables(party, qb, ws, B, gr)
    geo = (comp.N, comp.n, comp.ks, comp.ls)

    def level_vectors(slots):
        out = {}
        k16 = (B == 16 and gr.d == 64 and comp.n == 1 and comp.N % 16 == 0 and not _K16_OFF
               and all(t.is_contiguous() and t.data_ptr() % 16 == 0
                       for sl in slots.values() for t in sl["y"].values()))
        for side in ("x", "y"):
            # m is the same public value at P1 and P2 (honest joint session)
            srcs = [(rr, k, t) for rr, sl in sorted(slots.items()) for k, t in sl[side].items()
                    if not (rr == 2 and k == "m" and 1 in slots and "m" in slots[1][side])]
            dst = [empty((nb, gr.d)) for _ in srcs]
            for c0 in range(0, len(srcs), 4):          # wide blocks: <= 4 components per launch
                part, pdst = srcs[c0:c0 + 4], dst[c0:c0 + 4]
                if rows16:
                    xside = side == "x"
                    call("r3_vfy_mul16_line", int(xside), len(part), _ptrs([t for _, _, t in part]), comp.N,
                         ptr(qb[0]) if xside else None, ptr(rk if xside else kappa), gr.mod.lowterms_mask,
                         gr.d, _ptrs(pdst), gr.mask, stream())
                elif side == "x":
                    call("r3_vfy_line_b", B, len(part), _ptrs([t for _, _, t in part]), *geo, ptr(tabs),
                         nb * gr.d, B, gr.d, _ptrs(pdst), gr.mask, stream())
                elif k16:
                    # kappa_a y_(16j + a) as a K = 16 byte-limb GEMM per component
                    for (_, _, t), o in zip(part, pdst):
                        call("r3_gr_matmul_k16_tc", ptr(t), nb, ptr(kappa), ptr(o), gr.mask, stream())
                else:
                    call("r3_vfy_line_b_const", B, len(part), _ptrs([t for _, _, t in part]), *geo, ptr(kappa),
                         gr.d, _ptrs(pdst), gr.mask, stream())
            for (rr, k, _), o in zip(srcs, dst):
                out.setdefault(rr, {"x": {}, "y": {}})[side][k] = o
            if 2 in slots and "m" in slots[2][side] and "m" not in out.get(2, {}).get(side, {}):
                out.setdefault(2, {"x": {}, "y": {}})[side]["m"] = out[1][side]["m"]
        return out

    mine = {"x": comp.x, "y": comp.y}
    if _joint_ok(party):
        res = party.sess.joint(("lbvec", party.next_id("_joint.lbvec")), role, mine, level_vectors)
    else:
        res = level_vectors({role: mine})[role]
    return (_mval_from(res["x"], gr, role), _mval_from(res["y"], gr, role)), z, levels


def _base_tables(party, qb, ws: list, B: int, gr: Ring, tables: bool = True):
    """kappa_a = prod_{l < log2 B} w_(l+1)[bit l of a] (the level line weight
    of base element Bj + a) and the tables V_a[j] = pwB[j] (r^a kappa_a),
    a < B, built four at a time from one pass over pwB.  tables=False
    returns (None, kappa, r^a kappa_a) for the table-free d = 16 rows."""
    pwb, rpow = qb
    key = ("lbt", B, tables, gr.ell, gr.d, id(pwb), pwb.shape[0], tuple(_opened_key(party, w[1]) for w in ws))

    def build():
        kappa = None
        for lvl, w in enumerate(ws):
            f = torch.cat([w[(a >> lvl) & 1] for a in range(B)])
            kappa = f if kappa is None else grvec.gr_mul(kappa, f, gr.ell, gr.mod)
        rk = grvec.gr_mul(kappa, rpow, gr.ell, gr.mod)
        if not tables:
            return None, kappa.contiguous(), rk.contiguous()
        rows = pwb.shape[0]
        tabs = grvec.empty((B, rows, gr.d))
        for h in range(0, B, _TABLE_Q):
            grvec.rows_times_multi(pwb, [grvec.gr_mulmat(rk[a:a + 1], gr.mod) for a in range(h, h + _TABLE_Q)],
                                   rows, gr.ell, [tabs[a] for a in range(h, h + _TABLE_Q)])
        return tabs, kappa.contiguous()
    return _public(party, key, build)


def _joint_ok(party) -> bool:
    """Honest coop sessions may batch the three simulated parties' local
    kernels into one launch (Session.joint)."""
    from .transport import CoopRouter
    sess = party.sess
    return sess.joint_enabled and isinstance(sess.router, CoopRouter)


def _l2_tables(party, pw: torch.Tensor, dot_n: int, w1, ze2: torch.Tensor, gr: Ring):
    """kappa_a = w1_{a&1} w2_{a>>1} (w2 = (1 - ze_2, ze_2)) and the public
    tables V_a = pw_{(4j+a)} kappa_a (one row per block for multiplication
    logs; every power for dot logs)."""
    key = ("l2t", gr.ell, gr.d, id(pw), dot_n, _opened_key(party, ze2))

    def build():
        one = grvec.gr_const(1, gr.mod, gr.ell)
        w2 = (grvec.sub(one, ze2, gr.ell), ze2)
        kappa = torch.cat([grvec.gr_mul(w1[a & 1], w2[a >> 1], gr.ell, gr.mod) for a in range(4)])
        P = pw.shape[0]
        rows = (P + 3) // 4 if dot_n == 1 else P
        tabs = grvec.empty((4, rows, gr.d))
        for a in range(4):
            src = pw[a::4] if dot_n == 1 else pw
            if src.shape[0]:
                M = grvec.gr_mulmat(kappa[a:a + 1], gr.mod)
                grvec.rows_times(src, M, src.shape[0], gr.ell, out=tabs[a, :src.shape[0]])
            if src.shape[0] < rows:
                tabs[a, src.shape[0]:].zero_()      # only the rows past the log are padding
        return tabs, kappa, (4 if dot_n == 1 else dot_n), rows * gr.d
    return _public(party, key, build)


def _l2_tables_q4(party, q4, w1, ze2: torch.Tensor, gr: Ring):
    """_l2_tables for multiplication logs from the r^(4j) table:
    V_a[j] = pw[4j + a] kappa_a = pw4[j] (r^a kappa_a)."""
    pw4, rpow = q4
    key = ("l2t4", gr.ell, gr.d, id(pw4), pw4.shape[0], _opened_key(party, ze2))

    def build():
        one = grvec.gr_const(1, gr.mod, gr.ell)
        w2 = (grvec.sub(one, ze2, gr.ell), ze2)
        kappa = torch.cat([grvec.gr_mul(w1[a & 1], w2[a >> 1], gr.ell, gr.mod) for a in range(4)])
        rk = grvec.gr_mul(kappa, rpow, gr.ell, gr.mod)
        rows = pw4.shape[0]
        tabs = grvec.empty((4, rows, gr.d))        # every row is written below
        grvec.rows_times_multi(pw4, [grvec.gr_mulmat(rk[a:a + 1], gr.mod) for a in range(4)], rows, gr.ell,
                               [tabs[a] for a in range(4)])
        return tabs, kappa, 4, rows * gr.d
    return _public(party, key, build)


def _materialise(comp: _Compressed, pw: torch.Tensor, gr: Ring, role: int):
    """Dense lifted vectors (only needed when R == 0)."""
    def flat(t):
        return t.reshape(-1) if comp.n == 1 else t.transpose(0, 1).reshape(-1)
    pw_rep = pw if comp.n == 1 else pw.repeat_interleave(comp.n, dim=0)
    xo = {k: grvec.gr_scale_rows(flat(t).contiguous(), pw_rep, gr.ell) for k, t in comp.x.items()}
    yo = {k: grvec.gr_embed(flat(t).contiguous(), gr.mod) for k, t in comp.y.items()}
    return _mval_from(xo, gr, role), _mval_from(yo, gr, role)


# ---------------------------------------------------------------------------
# reference-shaped stages (public API)
# ---------------------------------------------------------------------------

def compress_mul_triples(party, xs: MVal, ys: MVal, zs: MVal, gr: Ring, chal: Challenges):
    """Pi_tran on a multiplication log: materialised (N, d) outputs."""
    r = _open_challenge(party, chal.r, "vfy.r")
    n = xs.lanes
    pw = _powers(party, r, n, gr)
    xl = _lift(xs, gr)
    xg = MVal(xl.mask._map(lambda a: grvec.gr_mul(a, pw, gr.ell, gr.mod)),
              None if xl.m is None else grvec.gr_mul(xl.m, pw, gr.ell, gr.mod))
    yg = _lift(ys, gr)
    zl = _lift(zs, gr)
    zg = _sum_lanes(MVal(zl.mask._map(lambda a: grvec.gr_mul(a, pw, gr.ell, gr.mod)),
                         None if zl.m is None else grvec.gr_mul(zl.m, pw, gr.ell, gr.mod)), gr)
    return xg, yg, zg


def consolidate_dot_triples(party, batches, gr: Ring, chal: Challenges):
    """Pi_bsv consolidation (verify.py:182-212), materialised."""
    r = _open_challenge(party, chal.r, "vfy.r")
    total = sum(b.lanes for b in batches)
    pw = _powers(party, r, total, gr)
    xs = ys = z_acc = None
    pos = 0
    for b in batches:
        p = pw[pos:pos + b.lanes]
        pos += b.lanes
        flat = lambda v: MVal(v.mask._map(lambda a: a.transpose(0, 1).reshape(-1, gr.d)),
                              None if v.m is None else v.m.transpose(0, 1).reshape(-1, gr.d))
        xf, yf = flat(_lift(b.xs, gr)), flat(_lift(b.ys, gr))
        p_rep = p.repeat_interleave(b.n, dim=0)
        xp = MVal(xf.mask._map(lambda a: grvec.gr_mul(a, p_rep, gr.ell, gr.mod)),
                  None if xf.m is None else grvec.gr_mul(xf.m, p_rep, gr.ell, gr.mod))
        zl = _lift(b.z, gr)
        zg = _sum_lanes(MVal(zl.mask._map(lambda a: grvec.gr_mul(a, p, gr.ell, gr.mod)),
                             None if zl.m is None else grvec.gr_mul(zl.m, p, gr.ell, gr.mod)), gr)
        xs = xp if xs is None else xs.concat(xp)
        ys = yf if ys is None else ys.concat(yf)
        z_acc = zg if z_acc is None else z_acc + zg
    return xs, ys, z_acc


class _Halves:
    """Even/odd rows of one dense (N, d) component as lazy linear operands.
    A zero lane appended to odd N (verify.py:220-222) is expressed by row
    validity, never materialised; f2 = 2 f1 - f0 and f1 - f0 are combined
    inside the kernels' operand loads."""

    def __init__(self, t: torch.Tensor):
        n = t.shape[0]
        self.ev, self.od = t[0::2], t[1::2]
        self.n0, self.n1 = (n + 1) // 2, n // 2

    def f0(self, c=1):
        return [(c, self.ev, self.n0)]

    def f1(self, c=1):
        return [(c, self.od, self.n1)]

    def f2(self, c=1):
        return [(2 * c, self.od, self.n1), (-c, self.ev, self.n0)]

    def d10(self):
        return [(1, self.od, self.n1), (-1, self.ev, self.n0)]


def _lin(terms):
    return grvec.lin(*[(c, t) for c, t, _ in terms], nvalid=[nv for _, _, nv in terms])


def _dotsum_terms(pairs, rows: int, gr: Ring) -> torch.Tensor:
    """sum over (F-terms, G-terms) of sum_i F_i (x) G_i, reduced: (1, d)."""
    acc = grvec.dotsum_acc(gr.d)
    for F, G in pairs:
        grvec.dotsum_add(acc, _lin(F), _lin(G), rows, gr.d)
    return grvec.reduce_poly(acc, gr.mod, gr.ell)


def _level_folds(role: int, X: dict, Y: dict, which: str, rows: int, gr: Ring) -> torch.Tensor:
    """The party's local fold of h(1) (which="f1") or h(2) (which="f2"):
    P0 sum F.total G.total; P1 -(F.m G.s1) - (G.m F.s1);
    P2 F.m (G.m - G.s2) - F.s2 G.m  (gates.dot_finish legs, gates.py:100-106)."""
    F = lambda c, k: getattr(X[c], which)(k)
    G = lambda c, k: getattr(Y[c], which)(k)
    if role == 0:
        pairs = [(F("total", 1), G("total", 1))]
    elif role == 1:
        pairs = [(F("m", -1), G("s1", 1)), (G("m", -1), F("s1", 1))]
    else:
        pairs = [(F("m", 1), G("m", 1) + G("s2", -1)), (F("s2", -1), G("m", 1))]
    return _dotsum_terms(pairs, rows, gr)


_JOINT16_MIN_ROWS = 1 << 14


def _level_folds_joint16(party, xt: dict, yt: dict, gr: Ring):
    """d = 16 dense-level folds of all three simulated parties at once
    (honest joint sessions): P1's and P2's four leg terms share one
    tensor-core pass (r3_vfy_level_fold16_tc), P0's single term a second,
    one-item-per-chunk pass.  Each party deposits only its own component arrays and
    takes only its own folds."""
    role = party.role
    names = ("total",) if role == 0 else ("m", "s1" if role == 1 else "s2")
    mine = {"x": [xt[k].contiguous() for k in names], "y": [yt[k].contiguous() for k in names]}

    return party.sess.joint(("fold16", party.next_id("_joint.fold16")), role, mine,
                            lambda slots: _folds16_all(slots, gr))


def _folds16_all(slots: dict, gr: Ring) -> dict:
    """The d = 16 tensor-core folds of all three parties (slots[r]["x"] /
    ["y"]: P0 [total], P1 / P2 [m, s1 / s2]): {r: (fold h1, fold h2)}."""
    N = slots[0]["x"][0].shape[0]
    acc_all = grvec.zeros((3, 2, 2 * gr.d - 1))
    accs = {r: acc_all[r] for r in range(3)}
    P = C.c_void_p
    xa, ya = slots[0]["x"][0], slots[0]["y"][0]
    # P0's single term: one y half, 1/8 of the MMA used -- still faster
    # than its CUDA-core fold
    call("r3_vfy_level_fold16_tc", 1, (C.c_int * 1)(0), (P * 1)(xa.data_ptr()), (P * 1)(ya.data_ptr()),
         (P * 1)(None), (C.c_int64 * 1)(1), (C.c_int64 * 1)(0), N,
         (P * 3)(accs[0][0].data_ptr(), None, None), (P * 3)(accs[0][1].data_ptr(), None, None), stream())
    (m1x, s1x), (m1y, s1y) = slots[1]["x"], slots[1]["y"]
    (m2x, s2x), (m2y, s2y) = slots[2]["x"], slots[2]["y"]
    # P1: -(m_x s_y1) - (s_x1 m_y);  P2: m_x (m_y - s_y2) - s_x2 m_y
    terms = [(1, m1x, s1y, None, -1, 0), (1, s1x, m1y, None, -1, 0),
             (2, m2x, m2y, s2y, 1, -1), (2, s2x, m2y, None, -1, 0)]
    party_ids = (C.c_int * 4)(*[t[0] for t in terms])
    xs = (P * 4)(*[t[1].data_ptr() for t in terms])
    y0 = (P * 4)(*[t[2].data_ptr() for t in terms])
    y1 = (P * 4)(*[None if t[3] is None else t[3].data_ptr() for t in terms])
    c0 = (C.c_int64 * 4)(*[t[4] for t in terms])
    c1 = (C.c_int64 * 4)(*[t[5] for t in terms])
    a1 = (P * 3)(None, accs[1][0].data_ptr(), accs[2][0].data_ptr())
    a2 = (P * 3)(None, accs[1][1].data_ptr(), accs[2][1].data_ptr())
    call("r3_vfy_level_fold16_tc", 4, party_ids, xs, y0, y1, c0, c1, N, a1, a2, stream())
    red = grvec.reduce_poly_rows(acc_all, gr.mod, gr.ell)   # (6, d): one launch
    return {r: (red[2 * r:2 * r + 1], red[2 * r + 1:2 * r + 2]) for r in range(3)}


def _level_folds_fused(role: int, xt: dict, yt: dict, gr: Ring, party=None):
    """Both folds of one party in one pass (r3_vfy_level_fold) when the
    component arrays are dense (N, d) rows; None -> use the dot-sum path."""
    if gr.d not in (16, 32, 64):
        return None
    if (party is not None and gr.d == 16 and _joint_ok(party)
            and next(iter(xt.values())).shape[0] >= _JOINT16_MIN_ROWS):
        return _level_folds_joint16(party, xt, yt, gr)
    if role == 0:
        names = ("total", None)
    else:
        names = ("m", "s1" if role == 1 else "s2")
    arrs = []
    for side in (xt, yt):
        for nm in names:
            t = None if nm is None else side.get(nm)
            if nm is not None and (t is None or not t.is_contiguous()):
                return None
            arrs.append(t)
    xa, xb, ya, yb = arrs
    N = xa.shape[0]
    acc = grvec.zeros((2, 2 * gr.d - 1))
    call("r3_vfy_level_fold", role, ptr(xa), ptr(xb), ptr(ya), ptr(yb), N, gr.d,
         ptr(acc[0]), ptr(acc[1]), stream())
    red = grvec.reduce_poly_rows(acc, gr.mod, gr.ell)
    return red[0:1], red[1:2]


def _line_eval(H: _Halves, Ms, gr: Ring) -> torch.Tensor:
    """f0 + (f1 - f0) * zeta (verify.py:239) = f0 . M(1 - zeta) + f1 . M(zeta):
    one K-concatenated contraction on the tensor cores for d = 64 / 16; the
    CUDA core form rows . M(zeta) + f0 otherwise."""
    M_one_m, M_z = Ms
    if gr.d in (16, 64):
        return grvec.rows_times(H.ev, M_one_m, H.n0, gr.ell, P1=H.od, M1=M_z,
                                nvalid=(H.n0, H.n1))
    return grvec.gr_matmul(_lin(H.d10()), M_z, H.n0, gr.d, gr.ell, C_add=_lin(H.f0()))


def _rdim_joint_ok(party, xs: MVal, gr: Ring) -> bool:
    if gr.d not in (16, 64) or not _joint_ok(party):
        return False
    return _rdim_shapes_ok(party, xs)


def _rdim_shapes_ok(party, xs: MVal) -> bool:
    """The honest tail shapes every party can decide alone: P0 holds only
    the mask sums of its vectors, P1 / P2 their half and m."""
    if party.role == 0:
        return xs.mask.total is not None and xs.mask.s1 is None
    return xs.m is not None


def _check_joint(sess, gr: Ring, slots: dict):
    """check_inner_product (Pi_vdot, verify.py:244-263) for all three parties
    in one rendezvous (honest joint sessions): the x' = alpha x gate
    (vfy.amul, n lanes), the vfy.dot gate of the n + 1 pairs
    ((x', alpha), (y, -z)) and the opening of delta (style "aux"), with every
    party's draws, messages (labels, classes, per-sender order) and values
    as in gate-by-gate execution.  Returns the zero test's device count."""
    P = sess.parties
    ell, d, mod = gr.ell, gr.d, gr.mod
    (x0, y0, z0, a0), (x1, y1, z1, a1), (x2, y2, z2, a2) = (slots[r] for r in range(3))
    n = x0.mask.total.shape[0]
    X0, X1s, X1m, X2s, X2m = x0.mask.total, x1.mask.s1, x1.m, x2.mask.s2, x1.m
    As1, As2, At, Am = a0.mask.s1, a0.mask.s2, a0.mask.total, a1.m
    # -- gate vfy.amul (lanes n): draws in stream order per party
    gid1 = [p.next_id("vfy.amul") for p in P]
    d01 = P[0].prg("01", "sha").draw_gr(2 * n, ell, mod)     # om.s1 (n), g.s1 (n)
    d02 = P[0].prg("02", "sha").draw_gr(n, ell, mod)         # om.s2
    P[1].prg("01", "sha").draw_gr(2 * n, ell, mod)
    P[2].prg("02", "sha").draw_gr(n, ell, mod)
    om_s1, g_s1, om_s2 = d01[:n], d01[n:], d02
    om_tot = grvec.add(om_s1, om_s2, ell)
    g_s2 = grvec.sub(grvec.add(grvec.gr_mul(X0, At, ell, mod), om_tot, ell), g_s1, ell)   # Gamma - s1
    # P1: -(x.m alpha.s1) - (alpha.m x.s1) + Gamma.s1; P2: x.m (alpha.m - alpha.s2) - alpha.m x.s2 + Gamma.s2
    leg1 = grvec.sub3(g_s1, grvec.gr_mul(X1m, As1, ell, mod), grvec.gr_mul(X1s, Am, ell, mod), ell)
    leg2 = grvec.sub(grvec.add(grvec.gr_mul(X2m, grvec.sub(Am, As2, ell), ell, mod), g_s2, ell),
                     grvec.gr_mul(X2s, Am, ell, mod), ell)
    mx = grvec.add(leg1, leg2, ell)
    P[0].send(2, f"sha.vfy.amul.gamma.{gid1[0]}", g_s2, gr, cls=OFFLINE, site="vfy.amul.gamma", gate=gid1[0])
    P[2].recv(0, f"sha.vfy.amul.gamma.{gid1[2]}", gr, n)
    P[1].send(2, f"vfy.amul.mz.{gid1[1]}.leg1", leg1, gr, cls=PAYLOAD, site="vfy.amul.mz", gate=gid1[1])
    P[2].send(1, f"vfy.amul.mz.{gid1[2]}.leg2", leg2, gr, cls=AUX, site="vfy.amul.mz", gate=gid1[2])
    P[1].recv(2, f"vfy.amul.mz.{gid1[1]}.leg2", gr, n)
    P[2].recv(1, f"vfy.amul.mz.{gid1[2]}.leg1", gr, n)
    # -- gate vfy.dot over the n + 1 pairs (x', alpha) . (y, -z)
    cat = lambda a, b: torch.cat([a, b])
    pxt, pyt = cat(om_tot, At), cat(y0.mask.total, grvec.vneg(z0.mask.total, ell))
    px1, py1 = cat(om_s1, As1), cat(y1.mask.s1, grvec.vneg(z1.mask.s1, ell))
    px2, py2 = cat(om_s2, As2), cat(y2.mask.s2, grvec.vneg(z2.mask.s2, ell))
    pxm, pym = cat(mx, Am), cat(y1.m, grvec.vneg(z1.m, ell))
    rows = n + 1
    acc = grvec.zeros((3, 2 * d - 1))
    L = grvec.lin
    grvec.dotsum_add(acc[0], L((1, pxt)), L((1, pyt)), rows, d)                     # P0 cross
    grvec.dotsum_add(acc[1], L((-1, pxm)), L((1, py1)), rows, d)                    # P1 legs
    grvec.dotsum_add(acc[1], L((-1, pym)), L((1, px1)), rows, d)
    grvec.dotsum_add(acc[2], L((1, pxm)), L((1, pym), (-1, py2)), rows, d)          # P2 legs
    grvec.dotsum_add(acc[2], L((-1, px2)), L((1, pym)), rows, d)
    red = grvec.reduce_poly_rows(acc, mod, ell)
    gid2 = [p.next_id("vfy.dot") for p in P]
    e01 = P[0].prg("01", "sha").draw_gr(2, ell, mod)          # om2.s1, g2.s1
    e02 = P[0].prg("02", "sha").draw_gr(1, ell, mod)          # om2.s2
    P[1].prg("01", "sha").draw_gr(2, ell, mod)
    P[2].prg("02", "sha").draw_gr(1, ell, mod)
    om2_s1, g2_s1, om2_s2 = e01[0:1], e01[1:2], e02
    om2_tot = grvec.add(om2_s1, om2_s2, ell)
    g2_s2 = grvec.sub(grvec.add(red[0:1], om2_tot, ell), g2_s1, ell)
    l1 = grvec.add(red[1:2], g2_s1, ell)
    l2 = grvec.add(red[2:3], g2_s2, ell)
    dm = grvec.add(l1, l2, ell)
    P[0].send(2, f"sha.vfy.dot.gamma.{gid2[0]}", g2_s2, gr, cls=OFFLINE, site="vfy.dot.gamma", gate=gid2[0])
    P[2].recv(0, f"sha.vfy.dot.gamma.{gid2[2]}", gr, 1)
    P[1].send(2, f"vfy.dot.mz.{gid2[1]}.leg1", l1, gr, cls=PAYLOAD, site="vfy.dot.mz", gate=gid2[1])
    P[2].send(1, f"vfy.dot.mz.{gid2[2]}.leg2", l2, gr, cls=PAYLOAD, site="vfy.dot.mz", gate=gid2[2])
    P[1].recv(2, f"vfy.dot.mz.{gid2[1]}.leg2", gr, 1)
    P[2].recv(1, f"vfy.dot.mz.{gid2[2]}.leg1", gr, 1)
    # -- open delta (sharing.rec, style "aux": every leg auxiliary)
    tags = [f"vfy.delta#{p.next_id('rec')}" for p in P]
    T = lambda r, leg: f"rec.{tags[r]}.{leg}"
    P[0].send(2, T(0, "r1"), om2_s1, gr, cls=AUX)
    P[0].send(1, T(0, "r2"), om2_s2, gr, cls=AUX)
    P[1].send(0, T(1, "m"), dm, gr, cls=AUX)
    P[1].send_digest(2, T(1, "r1"), om2_s1, gr)
    P[2].send_digest(0, T(2, "m"), dm, gr)
    P[2].send_digest(1, T(2, "r2"), om2_s2, gr)
    m0 = P[0].recv(1, T(0, "m"), gr, 1)
    P[0].check_digest(2, T(0, "m"), m0, gr, f"rec {tags[0]} m")
    s2_1 = P[1].recv(0, T(1, "r2"), gr, 1)
    P[1].check_digest(2, T(1, "r2"), s2_1, gr, f"rec {tags[1]} r2")
    s1_2 = P[2].recv(0, T(2, "r1"), gr, 1)
    P[2].check_digest(1, T(2, "r1"), s1_2, gr, f"rec {tags[2]} r1")
    bad = grvec.count_nonequal(grvec.sub3(dm, om2_s1, om2_s2, ell))
    return {0: bad, 1: bad, 2: bad}


def _reduce_dimension_joint(party, xs: MVal, ys: MVal, z: MVal, gr: Ring, zeta: MVal):
    """reduce_dimension of all three simulated parties in ONE rendezvous
    (honest joint sessions, d = 64 / 16): every party's folds, the reduction
    round (_round_joint) and every line evaluation of the level (one
    multi-job tensor-core launch; m's evaluations once for P1 and P2).
    Local work and messages are the reference's; the round barrier follows
    the rendezvous as it follows the opening in reduce_dimension."""
    key = ("rdim", party.next_id("_joint.rdim"))
    out = party.sess.joint(key, party.role, (xs, ys, z, zeta), lambda slots: _rdim_compute(party.sess, gr, slots))
    party.round_barrier()
    return out


def _rdim_compute(sess, gr: Ring, slots: dict) -> dict:
    (x0, y0, z0, t0), (x1, y1, z1, t1), (x2, y2, z2, t2) = (slots[r] for r in range(3))
    comps = {0: (("total", x0.mask.total, y0.mask.total),),
             1: (("m", x1.m, y1.m), ("s1", x1.mask.s1, y1.mask.s1)),
             2: (("m", x2.m, y2.m), ("s2", x2.mask.s2, y2.mask.s2))}
    n = x0.mask.total.shape[0]
    rows = (n + 1) // 2
    d = gr.d
    if d == 16 and n >= _JOINT16_MIN_ROWS:
        folds = _folds16_all({r: {"x": [c[1].contiguous() for c in comps[r]],
                                  "y": [c[2].contiguous() for c in comps[r]]} for r in range(3)}, gr)
    elif d == 64 and (n + 1) // 2 >= 4096:           # the tensor-core size range of r3_vfy_level_fold
        # every party's terms in one tensor-core launch (m read once for P1
        # and P2), one reduction
        acc = empty((3, 2, 2 * d - 1))
        cc = lambda t: t.contiguous()
        Pp = C.c_void_p * 3
        call("r3_vfy_level_fold_joint", ptr(cc(x0.mask.total)), ptr(cc(y0.mask.total)), ptr(cc(x1.m)), ptr(cc(y1.m)),
             ptr(cc(x1.mask.s1)), ptr(cc(y1.mask.s1)), ptr(cc(x2.mask.s2)), ptr(cc(y2.mask.s2)), n,
             Pp(*[ptr(acc[r, 0]) for r in range(3)]), Pp(*[ptr(acc[r, 1]) for r in range(3)]), stream())
        red = grvec.reduce_poly_rows(acc, gr.mod, gr.ell)
        folds = {r: (red[2 * r:2 * r + 1], red[2 * r + 1:2 * r + 2]) for r in range(3)}
    else:
        # one r3_vfy_level_fold per party into one accumulator block, one reduction
        acc = grvec.zeros((3, 2, 2 * d - 1))
        for r in range(3):
            c = comps[r]
            xa, ya = c[0][1].contiguous(), c[0][2].contiguous()
            xb = c[1][1].contiguous() if len(c) > 1 else None
            yb = c[1][2].contiguous() if len(c) > 1 else None
            call("r3_vfy_level_fold", r, ptr(xa), ptr(xb), ptr(ya), ptr(yb), n, d,
                 ptr(acc[r, 0]), ptr(acc[r, 1]), stream())
        red = grvec.reduce_poly_rows(acc, gr.mod, gr.ell)
        folds = {r: (red[2 * r:2 * r + 1], red[2 * r + 1:2 * r + 2]) for r in range(3)}
    rnd = _round_joint(sess, gr, rows, {r: (folds[r][0], folds[r][1], slots[r][2], slots[r][3]) for r in range(3)})
    q = rnd[0][2]
    # every component's line evaluation in one launch: P0 total, P1 s1,
    # P2 s2 (x and y), m once
    srcs = [(0, "total", "x", x0.mask.total), (0, "total", "y", y0.mask.total),
            (1, "s1", "x", x1.mask.s1), (1, "s1", "y", y1.mask.s1),
            (2, "s2", "x", x2.mask.s2), (2, "s2", "y", y2.mask.s2),
            (1, "m", "x", x1.m), (1, "m", "y", y1.m)]
    hs = [_Halves(t) for *_, t in srcs]
    res = grvec.rows_times2_batch([(H.ev, H.od, H.n0, H.n1) for H in hs], q.M_one_m, q.M_ze, gr.ell)
    o = {(r, k, side): v for (r, k, side, _), v in zip(srcs, res)}
    mx, my = o[(1, "m", "x")], o[(1, "m", "y")]
    out = {}
    for r, (xs, ys) in ((0, (x0, y0)), (1, (x1, y1)), (2, (x2, y2))):
        k = ("total", "s1", "s2")[r]
        m_x, m_y = (None, None) if r == 0 else (mx, my)
        xo = MVal(AShare(gr, r, **{k: o[(r, k, "x")]}, p0_halves=xs.mask.p0_halves), m_x)
        yo = MVal(AShare(gr, r, **{k: o[(r, k, "y")]}, p0_halves=ys.mask.p0_halves), m_y)
        out[r] = (xo, yo, rnd[r][0])
    return out


def reduce_dimension(party, xs: MVal, ys: MVal, z: MVal, gr: Ring, zeta: MVal):
    """Halve the triple (verify.py:215-241): pad odd lengths with a zero lane,
    h(1), h(2) by inner products, h(0) = z - h(1), evaluate at 2*zeta."""
    if _rdim_joint_ok(party, xs, gr):
        return _reduce_dimension_joint(party, xs, ys, z, gr, zeta)
    role = party.role
    names = [k for k in ("s1", "s2", "total") if getattr(xs.mask, k) is not None]
    X = {k: _Halves(getattr(xs.mask, k)) for k in names}
    Y = {k: _Halves(getattr(ys.mask, k)) for k in names}
    if xs.m is not None:
        X["m"], Y["m"] = _Halves(xs.m), _Halves(ys.m)
    rows = next(iter(X.values())).n0
    small = gr.d < 8
    if small:  # degrees 1..4: generic kernels, materialised halves
        return _reduce_dimension_small(party, xs, ys, z, gr, zeta)
    xt = {k: getattr(xs.mask, k) for k in names}
    yt = {k: getattr(ys.mask, k) for k in names}
    if xs.m is not None:
        xt["m"], yt["m"] = xs.m, ys.m
    fused = _level_folds_fused(role, xt, yt, gr, party)
    if fused is not None:
        fold1, fold2 = fused
    else:
        fold1 = _level_folds(role, X, Y, "f1", rows, gr)
        fold2 = _level_folds(role, X, Y, "f2", rows, gr)
    z_out, ze, q = _reduction_round(party, gr, rows, fold1, fold2, z, zeta)
    Ms = (q.M_one_m if gr.d in (16, 64) else None, q.M_ze)
    if gr.d in (16, 64):
        xo, yo, mx, my = _level_line_evals(party, X, Y, names, Ms, gr)
        mk = lambda o, m, v: MVal(AShare(gr, role, **o, p0_halves=v.mask.p0_halves), m)
        return mk(xo, mx, xs), mk(yo, my, ys), z_out
    out = lambda V, k: _line_eval(V[k], Ms, gr)
    mk = lambda V, v: MVal(AShare(gr, role, **{k: out(V, k) for k in names},
                                  p0_halves=v.mask.p0_halves),
                           _shared_m(party, lambda: out(V, "m")) if "m" in V else None)
    return mk(X, xs), mk(Y, ys), z_out


def _level_line_evals(party, X: dict, Y: dict, names: list, Ms, gr: Ring):
    """Every line evaluation f0 . M(1 - zeta) + f1 . M(zeta) (verify.py:239-240)
    of one party's reduction level in one tensor-core launch (d = 64): its
    mask components of x and y, plus the m components when this party is
    the one that builds them (the _shared_m rule: in honest joint sessions
    the first of P1 / P2 to arrive computes m's evaluations, the other
    takes the same tensors)."""
    jobs = [X[k] for k in names] + [Y[k] for k in names]
    mx = my = None
    key = None
    build_m = "m" in X
    if build_m and party.role != 0 and _joint_ok(party):
        key = ("m", party.next_id("_shared_m"))
        memo = party.sess.shared_m
        if key in memo:
            mx, my = memo.pop(key)
            build_m = False
    if build_m:
        jobs += [X["m"], Y["m"]]
    res = grvec.rows_times2_batch([(H.ev, H.od, H.n0, H.n1) for H in jobs], Ms[0], Ms[1], gr.ell)
    n = len(names)
    xo, yo = dict(zip(names, res[:n])), dict(zip(names, res[n:2 * n]))
    if build_m:
        mx, my = res[2 * n], res[2 * n + 1]
        if key is not None:
            party.sess.shared_m[key] = (mx, my)
    return xo, yo, mx, my


def _reduce_dimension_small(party, xs, ys, z, gr, zeta):
    """Reference-shaped reduction for tiny degrees (d < 8)."""
    if xs.lanes % 2 == 1:
        pad = _zero_lanes(party, gr, 1)
        xs, ys = xs.concat(pad), ys.concat(pad)
    f0, f1 = xs.take(slice(0, None, 2)), xs.take(slice(1, None, 2))
    g0, g1 = ys.take(slice(0, None, 2)), ys.take(slice(1, None, 2))
    f2 = f1.scale_pub(2) - f0
    g2 = g1.scale_pub(2) - g0
    h1 = _gr_dot(party, f1, g1, gr)
    h2 = _gr_dot(party, f2, g2, gr)
    ze = _open_challenge(party, zeta.scale_pub(2), "vfy.zeta")
    z_out = _recombine(party, z, h1, h2, _quad(party, ze, gr), gr)
    xs_out = f0 + (f1 - f0).scale_gr(ze)
    ys_out = g0 + (g1 - g0).scale_gr(ze)
    return xs_out, ys_out, z_out


def check_inner_product(party, xs: MVal, ys: MVal, z: MVal, gr: Ring, alpha: MVal) -> bool:
    """Pi_vdot (verify.py:244-263): x' = alpha * x, fold (alpha, -z) in as
    the last pair, open the combination, accept iff it is zero."""
    if gr.mod is not None and _joint_ok(party) and _rdim_shapes_ok(party, xs):
        key = ("check", party.next_id("_joint.check"))
        bad = party.sess.joint(key, party.role, (xs, ys, z, alpha),
                               lambda slots: _check_joint(party.sess, gr, slots))
        party.round_barrier()
        if getattr(party, "_deferred_verdicts", None) is not None:
            return bad
        return int(bad.item()) == 0
    n = xs.lanes
    bcast = lambda a: a.expand((n,) + tuple(a.shape[1:]))
    alpha_n = MVal(alpha.mask._map(bcast), None if alpha.m is None else bcast(alpha.m), alpha.sealed)
    unsq = lambda v: MVal(v.mask._map(lambda a: a[None]), None if v.m is None else v.m[None], v.sealed)
    gate = dot_prepare(party, unsq(xs).mask, unsq(alpha_n).mask, lanes=n, kind="vfy.amul",
                       gamma_cls=OFFLINE)
    xprime = dot_finish(party, gate, unsq(xs), unsq(alpha_n), log=False, leg2_cls=AUX)
    pairs_x = xprime.concat(alpha)
    pairs_y = ys.concat(-z)
    delta = _gr_dot(party, pairs_x, pairs_y, gr)
    opened = rec(party, delta, "vfy.delta", style="aux")
    party.round_barrier()
    bad = grvec.count_nonequal(opened)
    if getattr(party, "_deferred_verdicts", None) is not None:
        return bad            # verify_session reads every log's count at its end
    return int(bad.item()) == 0


# ---------------------------------------------------------------------------
# drivers
# ---------------------------------------------------------------------------

def _cat_mvals(vals: list, dim: int = 0) -> MVal:
    """One torch.cat per field for the whole list (MVal.concat / _map
    semantics: a field survives only if every view has it)."""
    if len(vals) == 1:
        return vals[0]
    first = vals[0].mask
    fields = {}
    for f in ("s1", "s2", "total"):
        parts = [getattr(v.mask, f) for v in vals]
        fields[f] = None if any(t is None for t in parts) else torch.cat(parts, dim=dim)
    mask = AShare(first.ring, first.role, p0_halves=all(v.mask.p0_halves for v in vals), **fields)
    ms = [v.m for v in vals]
    return MVal(mask, None if ms[0] is None else torch.cat(ms, dim=dim))


def _concat_all(recs, pick):
    return _cat_mvals([pick(r) for r in recs])


def _verify_tail(party, xs, ys, z, gr, ctx: Challenges, R: int, start: int = 0) -> bool:
    if R > len(ctx.zetas):
        raise ConfigError(f"R={R} exceeds prepared challenge budget {len(ctx.zetas)}")
    for k in range(start, R):
        xs, ys, z = reduce_dimension(party, xs, ys, z, gr, ctx.zetas[k])
    return check_inner_product(party, xs, ys, z, gr, ctx.alpha)


def _require_ctx(party, key: str) -> Challenges:
    if party.verify_ctx is None or key not in party.verify_ctx:
        raise ConfigError("verification challenges were not prepared in the preprocessing phase")
    return party.verify_ctx[key]


def _require_kept_logs(party) -> None:
    if any(log.discard for log in party.logs.values()):
        raise HarnessError("gate logs were discarded (Party.discard_logs); nothing to verify")


def batch_verify_muls(party, base_ell: int, d: int, R: int, kind_key: str | None = None) -> bool:
    """Verify every logged multiplication of the given base ring."""
    return _verification_group(party, "mul", lambda: _batch_verify_muls(party, base_ell, d, R, kind_key))


def _batch_verify_muls(party, base_ell: int, d: int, R: int, kind_key: str | None) -> bool:
    _require_kept_logs(party)
    kind = "bool" if base_ell == 1 else "arith"
    log = party.logs[kind]
    if not log.muls:
        return True
    ctx = _require_ctx(party, kind_key or f"mul.{kind}")
    gr = Ring(base_ell, modulus_for_degree(d))
    if R > len(ctx.zetas):
        raise ConfigError(f"R={R} exceeds prepared challenge budget {len(ctx.zetas)}")
    xs = _concat_all(log.muls, lambda b: b.x)
    ys = _concat_all(log.muls, lambda b: b.y)
    zs = _concat_all(log.muls, lambda b: b.z)
    if len(log.muls) > 1:
        # the frozen log keeps the concatenated batch only (same values in
        # the same order), so the per-gate tensors are freed for the
        # verification's working set
        log.muls[:] = [MulBatchRec(xs, ys, zs, sum(b.lanes for b in log.muls))]
    comp = _compressed_from_log(xs, ys, party.role, 1)
    if _gf2_packed_ok(gr, R):
        return _verify_muls_gf2(party, comp, zs, gr, ctx, R)
    (xv, yv), z, done = _compress_reduce_first(party, comp, zs, comp.N, 1, gr, ctx, R)
    return _verify_tail(party, xv, yv, z, gr, ctx, R, start=done)


def _gf2_packed_ok(gr: Ring, R: int) -> bool:
    return gr.ell == 1 and 2 <= gr.d <= 32 and R >= 1


def _verify_muls_gf2(party, comp: _Compressed, zs: MVal, gr: Ring, chal: Challenges, R: int) -> bool:
    """Pi_tran + R x Pi_rd + Pi_vdot on a boolean multiplication log with the
    level vectors packed as GF(2^d) words (csrc/gf2.cu): level 0's folds
    and z power sums straight from the base bits (r3_gfv_base_fold), then
    every line evaluation fused with the next level's folds (r3_gfv_line);
    the last level is written in the reference's (n, d) layout for the
    check.  Every fold, message and verdict equals the reference's
    (characteristic 2: the same values as the (n, d) word arithmetic of
    verify.py:168-263)."""
    role = party.role
    names = list(comp.x)
    idx = {k: i for i, k in enumerate(names)}
    terms = [(idx[a], idx[b]) for _, a, b in _role_terms(role)]
    nc, nt = len(names), len(terms)
    tx = (C.c_int * nt)(*[t[0] for t in terms])
    ty = (C.c_int * nt)(*[t[1] for t in terms])
    zc = _components(zs, role)
    znames = list(zc)
    zc = {k: t.reshape(-1).contiguous() for k, t in zc.items()}
    d, f_low = gr.d, gr.mod.lowterms_mask
    P = C.c_void_p
    scratch = empty((4,))
    r = _open_challenge(party, chal.r, "vfy.r")
    folds = empty((2 + len(znames), d))
    call("r3_gfv_base_fold", nc, (P * nc)(*[ptr(comp.x[k]) for k in names]),
         (P * nc)(*[ptr(comp.y[k]) for k in names]), nt, tx, ty, len(znames),
         (P * 2)(*[ptr(zc[k]) for k in znames]), comp.N, ptr(r), d, f_low, ptr(folds), ptr(scratch), stream())
    z = _mval_from({k: folds[2 + i:3 + i] for i, k in enumerate(znames)}, gr, role)
    h1f, h2f = folds[0:1], folds[1:2]
    n = comp.N
    src = ([comp.x[k] for k in names], [comp.y[k] for k in names])
    for k in range(R):
        rows = (n + 1) // 2
        z, ze, _ = _reduction_round(party, gr, rows, h1f, h2f, z, chal.zetas[k])
        last = k == R - 1
        if last:
            outs = [empty((rows, d)) for _ in range(2 * nc)]
            nxt = None
        else:
            outs = [torch.empty(rows + 4, dtype=torch.int32, device=r.device) for _ in range(2 * nc)]
            nxt = empty((2, d))
        call("r3_gfv_line", 1 if k == 0 else 0, nc, (P * nc)(*[ptr(t) for t in src[0]]),
             (P * nc)(*[ptr(t) for t in src[1]]), n, ptr(r), ptr(ze), d, f_low, 1 if last else 0,
             (P * nc)(*[ptr(t) for t in outs[:nc]]), (P * nc)(*[ptr(t) for t in outs[nc:]]), nt, tx, ty,
             ptr(nxt), ptr(scratch), stream())
        src = (outs[:nc], outs[nc:])
        if nxt is not None:
            h1f, h2f = nxt[0:1], nxt[1:2]
        n = rows
    xs = _mval_from(dict(zip(names, src[0])), gr, role)
    ys = _mval_from(dict(zip(names, src[1])), gr, role)
    return check_inner_product(party, xs, ys, z, gr, chal.alpha)


def batch_verify_dots(party, base_ell: int, d: int, R: int) -> bool:
    """Verify every logged inner-product gate of the given base ring."""
    return _verification_group(party, "dot", lambda: _batch_verify_dots(party, base_ell, d, R))


def _batch_verify_dots(party, base_ell: int, d: int, R: int) -> bool:
    _require_kept_logs(party)
    kind = "bool" if base_ell == 1 else "arith"
    log = party.logs[kind]
    if not log.dots:
        return True
    ctx = _require_ctx(party, f"dot.{kind}")
    gr = Ring(base_ell, modulus_for_degree(d))
    if R > len(ctx.zetas):
        raise ConfigError(f"R={R} exceeds prepared challenge budget {len(ctx.zetas)}")
    if _structured_dots_ok(log.dots, gr):
        return _verify_dots_structured(party, log.dots, gr, ctx, R)
    ns = {b.n for b in log.dots}
    if len(ns) != 1:
        xs, ys, z = consolidate_dot_triples(party, log.dots, gr, ctx)
        return _verify_tail(party, xs, ys, z, gr, ctx, R)
    n = ns.pop()
    cat1 = lambda pick: _concat_lanes([pick(b) for b in log.dots])
    xs, ys, zs = cat1(lambda b: b.xs), cat1(lambda b: b.ys), _concat_all(log.dots, lambda b: b.z)
    comp = _compressed_from_log(xs, ys, party.role, n)
    (xv, yv), z, done = _compress_reduce_first(party, comp, zs, comp.N // n, 1, gr, ctx, R)
    return _verify_tail(party, xv, yv, z, gr, ctx, R, start=done)


# ---------------------------------------------------------------------------
# structured Pi_bsv for GEMM-form linear layers
# ---------------------------------------------------------------------------

class _FCBatch:
    """A GEMM-form dot batch (gates.MatmulBatchRec: lane l at GEMM index
    perm[l] = m N + n, dot index i < K) inside the consolidated vector of
    consolidate_dot_triples (verify.py:182-212): element (l, i) is
    r^(P + l) X[m, i] on the x side and W[i, n] on the y side.  For the
    linear layers the lane index splits additively, l = a(m) + c(n) (FC:
    a = mN, c = n; conv: a = b out P + p, c = oc P), so
        x[(l), i] = r^P r^a(m) r^c(n) X[m, i].
    Line evaluations act on the dot index only, so after k reductions (while
    K stays even, i.e. pairs never straddle a lane) the level vectors keep
    this form with X_k (M x K/2^k) and W_k (K/2^k x N) GR matrices, and
    every leg fold factorises exactly in GR:
        sum_{l,j} r^(P+l) X'[m,j] W'[j,n] = r^P sum_j (sum_m r^a(m) X'[m,j]) (sum_n r^c(n) W'[j,n]).
    The level costs (M + N) K_k GR products instead of M N K_k."""

    @staticmethod
    def split(rec):
        """(a, c) with lane l = a[m] + c[n] for every lane, or None."""
        M, N = rec.M, rec.N
        if rec.perm is None:
            dev = rec.z.m.device if rec.z.m is not None else rec.z.mask.total.device
            return torch.arange(M, device=dev) * N, torch.arange(N, device=dev)
        perm = rec.perm
        lanes = torch.empty_like(perm)
        lanes[perm] = torch.arange(perm.numel(), device=perm.device)   # gemm index -> lane
        L = lanes.reshape(M, N)
        a, c = L[:, 0] - L[0, 0], L[0, :]
        if not bool((L == a[:, None] + c[None, :]).all()):
            return None
        return a, c

    def __init__(self, rec, role: int, gr: Ring, P: int, pw: torch.Tensor, split):
        self.M, self.K, self.N, self.P = rec.M, rec.K, rec.N, P
        d = gr.d
        xc, yc = _components(rec.X, role), _components(rec.W, role)
        self.X = {k: grvec.gr_embed(t.reshape(-1).contiguous(), gr.mod).reshape(self.M, self.K, d)
                  for k, t in xc.items()}
        self.Wt = {k: grvec.gr_embed(t.reshape(self.K, self.N).t().contiguous().reshape(-1), gr.mod)
                   .reshape(self.N, self.K, d) for k, t in yc.items()}
        a, c = split
        self.RM = pw[a].contiguous()
        self.RN = pw[c].contiguous()
        self.rP = pw[P:P + 1]
        # lane l -> (m, n) and its power r^(P + l), for materialisation
        self.pw_lanes = pw[P:P + self.M * self.N]
        perm = rec.perm if rec.perm is not None else torch.arange(self.M * self.N, device=pw.device)
        self.lane_m, self.lane_n = perm // self.N, perm % self.N

    def length(self) -> int:
        return self.M * self.N * self.K

    def structured(self) -> bool:
        return self.K % 2 == 0

    @staticmethod
    def _weighted_colsum(R: torch.Tensor, A: torch.Tensor, gr: Ring) -> torch.Tensor:
        """out[j] = sum_r R[r] A[r, j] over GR: (J, d)."""
        rows, J, d = A.shape
        prod = grvec.gr_mul(A.reshape(rows * J, d), R.repeat_interleave(J, dim=0), gr.ell, gr.mod)
        return grvec.sum_axis0(prod.reshape(rows, J * d), gr.ell).reshape(J, d)

    def folds(self, role: int, gr: Ring):
        """(fold h(1), fold h(2)) of this batch for the party's leg terms."""
        def sides(T):
            out = {}
            for k, t in T.items():
                od, ev = t[:, 1::2], t[:, 0::2]
                t2 = grvec.sub(grvec.add(od, od, gr.ell), ev, gr.ell)
                out[k] = (od.contiguous(), t2)
            return out
        xs, ys = sides(self.X), sides(self.Wt)
        res = []
        for h in (0, 1):
            U = {k: self._weighted_colsum(self.RM, v[h], gr) for k, v in xs.items()}
            V = {k: self._weighted_colsum(self.RN, v[h], gr) for k, v in ys.items()}
            if role == 0:
                terms = [(U["total"], V["total"])]
            elif role == 1:
                terms = [(grvec.vneg(U["m"], gr.ell), V["s1"]), (grvec.vneg(U["s1"], gr.ell), V["m"])]
            else:
                terms = [(U["m"], grvec.sub(V["m"], V["s2"], gr.ell)), (grvec.vneg(U["s2"], gr.ell), V["m"])]
            acc = None
            for a, b in terms:
                t = grvec.gr_dot(a, b, gr.ell, gr.mod)
                acc = t if acc is None else grvec.add(acc, t, gr.ell)
            res.append(grvec.gr_mul(acc, self.rP, gr.ell, gr.mod))
        return res[0], res[1]

    def reduce(self, Ms, gr: Ring) -> None:
        d = gr.d
        half = lambda t, rows: _line_eval(_Halves(t.reshape(-1, d)), Ms, gr).reshape(rows, -1, d)
        self.X = {k: half(t, self.M) for k, t in self.X.items()}
        self.Wt = {k: half(t, self.N) for k, t in self.Wt.items()}
        self.K //= 2

    def materialise(self, gr: Ring):
        """The batch's level vectors in the reference layout (lane-major):
        x[(l, i)] = r^(P+l) X[m(l), i], y[(l, i)] = W[i, n(l)].  For d = 16 /
        64 the lane power is split, r^(P+l) = r^c(n) (r^P r^a(m)): the M K
        products X'' = r^(P+a(m)) X are formed once, then X'' times every
        n's multiplication matrix M(r^c(n)) is ONE byte-limb u64 GEMM on the
        tensor cores (X'' [M K x d] . [M(r^c(0)) | ... ] [d x N d], instead of
        M N K elementwise GR products), gathered into lane order."""
        K, d = self.K, gr.d
        yo = {k: t[self.lane_n].reshape(-1, d).contiguous() for k, t in self.Wt.items()}
        if d not in (16, 64):
            p_rep = self.pw_lanes.repeat_interleave(K, dim=0)
            xo = {k: grvec.gr_mul(t[self.lane_m].reshape(-1, d), p_rep, gr.ell, gr.mod) for k, t in self.X.items()}
            return xo, yo
        M, N = self.M, self.N
        R = M * K
        rpa = grvec.gr_mul(self.RM, self.rP, gr.ell, gr.mod).repeat_interleave(K, dim=0)    # (M K, d)
        # B = [M(r^c(0)) | ... | M(r^c(N-1))] as K-major byte-limb tiles, built
        # once per batch (the lane powers do not change across levels)
        Kp, Np = max(32, d), -(-(N * d) // 64) * 64
        bt = getattr(self, "_rn_tiles", None)
        if bt is None:
            # all N multiplication matrices in one product: row k of M(x) is
            # x t^k, so M(r^c(n))[k] = r^c(n) (x) t^k for the d monomials t^k
            eye = torch.eye(d, dtype=torch.int64, device=self.RN.device)
            mats = grvec.gr_mul(self.RN.repeat_interleave(d, dim=0), eye.repeat(N, 1), gr.ell, gr.mod)
            Bm = grvec.zeros((Kp, Np))
            Bm[:d, :N * d] = mats.view(N, d, d).permute(1, 0, 2).reshape(d, N * d)
            bt = self._rn_tiles = grvec.limb_tiles_b(Bm)
        Rp = -(-R // 128) * 128
        dev = rpa.device
        idx = ((self.lane_m[:, None] * K + torch.arange(K, device=dev)[None, :]) * (Np // d)
               + self.lane_n[:, None]).reshape(-1)
        xo = {}
        for k, t in self.X.items():
            A = grvec.zeros((Rp, Kp))
            A[:R, :d] = grvec.gr_mul(t.reshape(-1, d).contiguous(), rpa, gr.ell, gr.mod)   # r^(P+a(m)) X
            out = grvec.u64_gemm([(grvec.limb_tiles_a(A), bt, Kp)], Rp, Np, gr.ell)       # every n in one GEMM
            xo[k] = out.view(-1, d)[idx]
        return xo, yo

    def to_dense(self, gr: Ring) -> "_DenseBatch":
        xo, yo = self.materialise(gr)
        return _DenseBatch.from_arrays(xo, yo)


class _DenseBatch:
    """Any other dot batch (n, L) of the consolidated vector.  Level 0 is
    never lifted: its folds come straight from the base log
    (r3_vfy_l1_fold over the batch's power rows) and the first line
    evaluation writes the dense level-1 rows from the base shares and the
    public tables r^(P+l) (1 - ze), r^(P+l) ze (r3_vfy_l1_line_x / _y), as
    _compress_reduce_first does for a whole equal-n log."""

    @classmethod
    def from_arrays(cls, x: dict, y: dict) -> "_DenseBatch":
        obj = cls.__new__(cls)
        obj.x, obj.y, obj.base = x, y, None
        return obj

    def __init__(self, b, role: int, gr: Ring, P: int, pw: torch.Tensor):
        self.base = _compressed_from_log(b.xs, b.ys, role, b.n)
        self.pw = pw[P:P + b.lanes]
        self.x = self.y = None
        self.level = 0          # base-form levels: 0 (l1 folds), 1 (l2 folds from 16 accumulators)
        self.ze1 = None

    def length(self) -> int:
        if self.base is not None:
            return (self.base.N + self.level) >> self.level if self.level else self.base.N
        return next(iter(self.x.values())).shape[0]

    def structured(self) -> bool:
        return self.length() % 2 == 0

    def folds(self, role: int, gr: Ring, party=None):
        if self.base is not None and self.level == 0:
            return _l1_folds(party, self.base, self.pw, gr)
        if self.base is not None:
            # level 1 from the base log: 16 scalar-weighted power sums, then
            # the public weights of the level-1 line (vfy2.cu)
            comp = self.base
            terms = _role_terms(role)
            coef = (C.c_int64 * len(terms))(*[t[0] for t in terms])
            acc = empty((16, gr.d))
            call("r3_vfy_l2_fold", len(terms), coef, _ptrs([comp.x[t[1]] for t in terms]),
                 _ptrs([comp.y[t[2]] for t in terms]), comp.N, comp.n, comp.ks, comp.ls, ptr(self.pw),
                 gr.d, ptr(acc), stream())
            W1, W2, self.w1 = _l2_weights(party, self.ze1, gr)   # ze1 is the latest opening here
            fold = lambda W: _dotsum_terms([([(1, acc, 16)], [(1, W, 16)])], 16, gr)
            return fold(W1), fold(W2)
        fused = _level_folds_fused(role, self.x, self.y, gr, party)
        if fused is not None:
            return fused
        X = {k: _Halves(t) for k, t in self.x.items()}
        Y = {k: _Halves(t) for k, t in self.y.items()}
        rows = next(iter(X.values())).n0
        return _level_folds(role, X, Y, "f1", rows, gr), _level_folds(role, X, Y, "f2", rows, gr)

    def reduce(self, Ms, gr: Ring, party=None, ze=None) -> None:
        comp = self.base
        if comp is not None and self.level == 0 and comp.N % 4 == 0 and gr.d >= 8:
            self.ze1, self.level = ze, 1      # stay in base form for the next level
            return
        if comp is not None and self.level == 1:
            # level-2 rows straight from the base shares (r3_vfy_line_b)
            tabs, kappa, tq, stride = _l2_tables(party, self.pw, comp.n, self.w1, ze, gr)
            nb = (comp.N + 3) // 4
            xk, yk = list(comp.x), list(comp.y)
            self.x = {k: empty((nb, gr.d)) for k in xk}
            self.y = {k: empty((nb, gr.d)) for k in yk}
            geo = (comp.N, comp.n, comp.ks, comp.ls)
            call("r3_vfy_line_b", 4, len(xk), _ptrs([comp.x[k] for k in xk]), *geo, ptr(tabs), stride, tq,
                 gr.d, _ptrs([self.x[k] for k in xk]), gr.mask, stream())
            call("r3_vfy_line_b_const", 4, len(yk), _ptrs([comp.y[k] for k in yk]), *geo, ptr(kappa), gr.d,
                 _ptrs([self.y[k] for k in yk]), gr.mask, stream())
            self.base = None
            return
        if comp is not None:
            self._write_level1(party, gr, ze, _line_tables(party, None, self.pw, comp.n, ze, gr))
            return
        if gr.d in (16, 64):   # every component in one launch
            keys = [("x", k) for k in self.x] + [("y", k) for k in self.y]
            hs = [_Halves(getattr(self, v)[k]) for v, k in keys]
            res = grvec.rows_times2_batch([(H.ev, H.od, H.n0, H.n1) for H in hs], Ms[0], Ms[1], gr.ell)
            nx = len(self.x)
            self.x = dict(zip(self.x, res[:nx]))
            self.y = dict(zip(self.y, res[nx:]))
            return
        self.x = {k: _line_eval(_Halves(t), Ms, gr) for k, t in self.x.items()}
        self.y = {k: _line_eval(_Halves(t), Ms, gr) for k, t in self.y.items()}

    def _write_level1(self, party, gr: Ring, ze, tables) -> None:
        """Level-1 rows from the base shares and the tables r^(P+l) (1 - ze),
        r^(P+l) ze (r3_vfy_l1_line_x / _y)."""
        comp = self.base
        A, B, one_m = tables
        half = (comp.N + 1) // 2
        xk, yk = list(comp.x), list(comp.y)
        self.x = {k: empty((half, gr.d)) for k in xk}
        self.y = {k: empty((half, gr.d)) for k in yk}
        call("r3_vfy_l1_line_x", len(xk), _ptrs([comp.x[k] for k in xk]), comp.N, comp.n, comp.ks,
             comp.ls, ptr(A), ptr(B), comp.n, gr.d, _ptrs([self.x[k] for k in xk]), gr.mask, stream())
        call("r3_vfy_l1_line_y", len(yk), _ptrs([comp.y[k] for k in yk]), comp.N, comp.n, comp.ks,
             comp.ls, ptr(one_m), ptr(ze), gr.d, _ptrs([self.y[k] for k in yk]), gr.mask, stream())
        self.base = None

    def materialise(self, gr: Ring, party=None):
        if self.base is not None:
            if self.level == 1:
                # the loop stopped between the two base levels: write level 1
                # (tables built here, uncached: ze1 is not the latest opening)
                one = grvec.gr_const(1, gr.mod, gr.ell)
                one_m = grvec.sub(one, self.ze1, gr.ell)
                A = grvec.gr_mul(self.pw, one_m, gr.ell, gr.mod)
                B = grvec.gr_mul(self.pw, self.ze1, gr.ell, gr.mod)
                self._write_level1(party, gr, self.ze1, (A, B, one_m))
                return self.x, self.y
            return _materialise_dense(self.base, self.pw, gr)
        return self.x, self.y


class _Lane16Batch:
    """A dot batch (n, L) with n % 16 == 0 at d = 16 inside the structured
    dot verification (the edaBits inner products of every ReLU / MaxPool
    layer): its first four levels' folds are public-weight combinations of
    256 per-lane sums (r3_vfy_lane16_fold, as _reduce_lanes16 for a whole
    log), its level-4 rows come from the base shares (r3_vfy_lane16_line),
    and from there it continues as a dense batch (N/16 rows instead of the
    N/4 of _DenseBatch's base form)."""

    def __init__(self, b, role: int, gr: Ring, P: int, pw: torch.Tensor):
        self.base = _compressed_from_log(b.xs, b.ys, role, b.n)
        self.pw = pw[P:P + b.lanes]
        self.level, self.ws, self.acc, self.dense = 0, [], None, None

    def length(self) -> int:
        return self.dense.length() if self.dense is not None else self.base.N >> self.level

    def structured(self) -> bool:
        return self.length() % 2 == 0

    def folds(self, role: int, gr: Ring, party=None):
        if self.dense is not None:
            return self.dense.folds(role, gr, party)
        comp = self.base
        if self.acc is None:
            terms = _role_terms(role)
            coef = (C.c_int64 * len(terms))(*[t[0] for t in terms])
            self.acc = empty((256, gr.d))
            call("r3_vfy_lane16_fold", len(terms), coef, _ptrs([comp.x[t[1]] for t in terms]),
                 _ptrs([comp.y[t[2]] for t in terms]), comp.N // comp.n, comp.n, ptr(self.pw), gr.d,
                 ptr(self.acc), stream())
        W1, W2 = _block_fold_weights(party, self.level, self.ws, 16, gr)
        fold = lambda W: _dotsum_terms([([(1, self.acc, 256)], [(1, W, 256)])], 256, gr)
        return fold(W1), fold(W2)

    def reduce(self, Ms, gr: Ring, party=None, ze=None, one_m=None) -> None:
        if self.dense is not None:
            self.dense.reduce(Ms, gr, party, ze)
            return
        self.ws.append((one_m, ze))
        self.level += 1
        if self.level < 4:
            return
        comp = self.base
        kappa = _lane_kappa(party, self.ws, gr)
        rows4 = comp.N // 16
        out = []
        for src, pow_side in ((comp.x, 1), (comp.y, 0)):
            keys = list(src)
            dst = {k: empty((rows4, gr.d)) for k in keys}
            call("r3_vfy_lane16_line", pow_side, len(keys), _ptrs([src[k] for k in keys]), comp.N // comp.n,
                 comp.n, ptr(self.pw) if pow_side else None, ptr(kappa), gr.mod.lowterms_mask, gr.d,
                 _ptrs([dst[k] for k in keys]), gr.mask, stream())
            out.append(dst)
        self.dense = _DenseBatch.from_arrays(out[0], out[1])
        self.base = self.acc = None

    def materialise(self, gr: Ring, party=None):
        if self.dense is None:
            raise HarnessError("lane16 dot batch materialised before its fourth level")
        return self.dense.materialise(gr, party)


def _materialise_dense(comp: "_Compressed", pw: torch.Tensor, gr: Ring):
    flat = lambda t: t.transpose(0, 1).contiguous().reshape(-1)
    p_rep = pw.repeat_interleave(comp.n, dim=0)
    xo = {k: grvec.gr_scale_rows(flat(t), p_rep, gr.ell) for k, t in comp.x.items()}
    yo = {k: grvec.gr_embed(flat(t), gr.mod) for k, t in comp.y.items()}
    return xo, yo


def _structured_dots_ok(batches, gr: Ring) -> bool:
    return gr.d >= 8 and any(isinstance(b, MatmulBatchRec) and b.K % 2 == 0 for b in batches)


def _verify_dots_structured(party, batches, gr: Ring, ctx: Challenges, R: int) -> bool:
    """Pi_bsv (verify.py:182-212) + R x Pi_rd + Pi_vdot with GEMM-form
    batches kept factorised (_FCBatch) while their dot dimension stays even;
    the remaining levels run on the materialised vector.  Every value
    (folds, messages, verdict) equals the reference's."""
    role = party.role
    r = _open_challenge(party, ctx.r, "vfy.r")
    total = sum(b.lanes for b in batches)
    pw = _powers(party, r, total, gr)
    # dot batches with lanes of 16k elements take the four-level base form
    # when every part's length keeps the loop structured to level 4
    lane16 = (not _LANES16_OFF and gr.d == 16 and R >= 4
              and all((b.lanes * b.n) % 16 == 0 for b in batches))
    parts, z_acc, pos = [], None, 0
    for b in batches:
        p = pw[pos:pos + b.lanes]
        zl = _lift(b.z, gr)
        zg = _sum_lanes(MVal(zl.mask._map(lambda a: grvec.gr_mul(a, p, gr.ell, gr.mod)),
                             None if zl.m is None else grvec.gr_mul(zl.m, p, gr.ell, gr.mod)), gr)
        z_acc = zg if z_acc is None else z_acc + zg
        # an odd dot dimension (conv 5x5 over one channel: K = 25) gains
        # nothing from the factorised form; its base-form dense batch never
        # lifts levels 0 and 1 (a quarter of the lifted level-0 bytes)
        split = _FCBatch.split(b) if isinstance(b, MatmulBatchRec) and b.K % 2 == 0 else None
        if split is not None:
            parts.append(_FCBatch(b, role, gr, pos, pw, split))
        elif lane16 and b.n % 16 == 0 and not isinstance(b, MatmulBatchRec):
            parts.append(_Lane16Batch(b, role, gr, pos, pw))
        else:
            parts.append(_DenseBatch(b, role, gr, pos, pw))
        pos += b.lanes
    z = z_acc
    k = 0
    while k < R:
        # a factorised batch whose dot dimension turned odd continues dense
        parts = [pt.to_dense(gr) if isinstance(pt, _FCBatch) and not pt.structured()
                 and pt.length() % 2 == 0 else pt for pt in parts]
        if not all(pt.structured() for pt in parts):
            break
        folds = [pt.folds(role, gr, party) if isinstance(pt, (_DenseBatch, _Lane16Batch)) else pt.folds(role, gr)
                 for pt in parts]
        fold1, fold2 = folds[0]
        for f1, f2 in folds[1:]:
            fold1, fold2 = grvec.add(fold1, f1, gr.ell), grvec.add(fold2, f2, gr.ell)
        rows = sum(pt.length() for pt in parts) // 2
        z, ze, q = _reduction_round(party, gr, rows, fold1, fold2, z, ctx.zetas[k])
        Ms = (q.M_one_m if gr.d in (16, 64) else None, q.M_ze)
        for pt in parts:
            if isinstance(pt, _Lane16Batch):
                pt.reduce(Ms, gr, party, ze, q.one_m)
            elif isinstance(pt, _DenseBatch):
                pt.reduce(Ms, gr, party, ze)
            else:
                pt.reduce(Ms, gr)
        k += 1
    mats = [pt.materialise(gr, party) if isinstance(pt, (_DenseBatch, _Lane16Batch)) else pt.materialise(gr)
            for pt in parts]
    xs = _mval_from({c: torch.cat([m[0][c] for m in mats]) for c in mats[0][0]}, gr, role)
    ys = _mval_from({c: torch.cat([m[1][c] for m in mats]) for c in mats[0][1]}, gr, role)
    del parts, mats
    return _verify_tail(party, xs, ys, z, gr, ctx, R, start=k)


def _concat_lanes(vals: list) -> MVal:
    """Concatenate (n, L_b) dot-log operands along the lane axis, which is the
    lane-major consolidation order of verify.py:195-201."""
    return _cat_mvals(vals, dim=1)


def verify_session(party, d: int, R: int | str = "auto", profile: str = "lan") -> dict:
    """Freeze the logs and run every applicable verification; per-log verdicts."""
    if party.phase is not Phase.POST:
        raise ConfigError("verification runs in the postprocessing phase")
    party.freeze_logs()
    _require_kept_logs(party)
    results: dict = {}
    # the logs' zero tests are read once at the end (one device -> host
    # synchronisation per session instead of one per log, so the host
    # enqueues the next log's verification while the GPU finishes this one)
    party._deferred_verdicts = True
    try:
        for kind, base_ell in (("arith", party.ell), ("bool", 1)):
            log = party.logs[kind]
            if log.muls:
                r_eff = pick_r(log.mul_count(), base_ell, d, profile) if R == "auto" else int(R)
                results[f"mul.{kind}"] = batch_verify_muls(party, base_ell, d, r_eff)
            if log.dots:
                n_total = sum(b.lanes * b.n for b in log.dots)
                r_eff = pick_r(n_total, base_ell, d, profile) if R == "auto" else int(R)
                results[f"dot.{kind}"] = batch_verify_dots(party, base_ell, d, r_eff)
    finally:
        party._deferred_verdicts = None
    return {k: v if isinstance(v, bool) else int(v.item()) == 0 for k, v in results.items()}
