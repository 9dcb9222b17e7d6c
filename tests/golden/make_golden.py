"""Generate the golden fixtures by running the READ-ONLY reference here.

Usage (build container only; /root/reference does not exist on GPU boxes):

    python tests/golden/make_golden.py [--only NAME]

For each case in tests/programs.py it runs the unmodified reference package
(`/root/reference/pkg/src/ring3pc`) under its deterministic "coop" engine --
with the thread-backed greenlet stand-in from oracle/refshim, because the
real greenlet wheel is not installed -- and records:

* every party's share components of the returned values (s1/s2/total/m);
* verdicts and opened values;
* the transcript counters, round counters and per-message
  (from, to, phase, label, nbytes, class) log;
* the SHA-256 of every message payload as sent (per sender, program order),
  captured by a Router subclass passed through Session(router_cls=...).

Outputs: tests/golden/<case>.npz (arrays + a JSON "meta" entry).  Nothing in
the reference tree is modified.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"

sys.path.insert(0, os.path.join(REPO, "oracle", "refshim"))
sys.path.insert(0, REF_SRC)
sys.path.insert(0, os.path.join(REPO, "tests"))

import ring3pc  # noqa: E402  (the reference)
from ring3pc import sharing as ref_sharing, transport as ref_transport  # noqa: E402
from ring3pc.runtime import Session  # noqa: E402

import programs  # noqa: E402


class RecordingRouter(ref_transport.CoopRouter):
    def __init__(self, transcript):
        super().__init__(transcript)
        self.payload_log = []

    def send(self, frm, to, phase, label, payload, cls="payload", count_bytes=None):
        self.payload_log.append((frm, to, phase.value, label, cls,
                                 hashlib.sha256(payload).hexdigest()))
        return super().send(frm, to, phase, label, payload, cls, count_bytes)


def _arr(a):
    return None if a is None else np.asarray(a, dtype=np.uint64)


def flatten_result(role: int, res, out: dict, prefix: str):
    """Store share components / arrays / verdicts of one party's result."""
    if isinstance(res, dict):
        for k, v in res.items():
            flatten_result(role, v, out, f"{prefix}.{k}" if prefix else k)
        return
    if isinstance(res, ref_sharing.MVal):
        for name, arr in (("m", res.m), ("s1", res.mask.s1), ("s2", res.mask.s2),
                          ("total", res.mask.total)):
            if arr is not None:
                out["arrays"][f"p{role}.{prefix}.{name}"] = _arr(arr)
        return
    if isinstance(res, (bool, np.bool_)):
        out["scalars"][f"p{role}.{prefix}"] = bool(res)
        return
    if isinstance(res, np.ndarray):
        out["arrays"][f"p{role}.{prefix}"] = _arr(res)
        return
    if res is None:
        return
    raise TypeError(f"unhandled result type {type(res)} at {prefix}")


def array_digest(a) -> str:
    """SHA-256 of a uint64 array's little-endian words (C order); the same
    function is applied to the GPU outputs by tests/test_gpu_golden_scale.py."""
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u8").tobytes()).hexdigest()


def run_case(name, prog_name, args, kwargs, sess_kw, injection=None, hashed=False):
    progs = programs.build("ring3pc")
    prog = getattr(progs, prog_name)
    adv = None
    if injection is not None:
        site, who, delta, gate, lane = injection
        adv = ref_transport.AdversaryConfig(
            corrupted=who,
            injections=[ref_transport.Injection(site, delta=delta, gate=gate, lane=lane)])
    sess = Session(seed=sess_kw.get("seed", 0), ell=sess_kw.get("ell", 64),
                   adversary=adv, keep_messages=True, engine="coop",
                   router_cls=RecordingRouter)
    out = {"arrays": {}, "scalars": {}}
    status = "ok"
    t0 = time.perf_counter()
    try:
        res = sess.run(lambda party: prog(party, *args, **kwargs))
        for role in range(3):
            flatten_result(role, res[role], out, "")
    except ref_transport.AbortError as e:
        status = f"abort:P{e.party}"
    dt = time.perf_counter() - t0
    tr = sess.transcript
    meta = {
        "name": name, "program": prog_name, "status": status,
        "session": sess_kw, "injection": injection,
        "counters": sorted([[f, t, p.value, c, n] for (f, t, p, c), n in tr.counters.items()]),
        "rounds": {p.value: n for p, n in tr.rounds.items()},
        "messages": [[f, t, p.value, lab, nb, c] for (f, t, p, lab, nb, c) in tr.messages],
        "payloads": sess.router.payload_log,
        "scalars": out["scalars"],
        "ref_seconds": dt,
    }
    arrays = dict(out["arrays"])
    target = HERE
    if hashed:
        # config-scale cases: one digest + shape per array keeps the fixture small
        meta["array_sha256"] = {k: [array_digest(v), list(v.shape)] for k, v in arrays.items()}
        arrays = {}
        target = os.path.join(HERE, "scale")
        os.makedirs(target, exist_ok=True)
    # program inputs (so the GPU tests need nothing but this file)
    for i, a in enumerate(args):
        if isinstance(a, np.ndarray):
            arrays[f"arg{i}"] = a.astype(np.uint64)
    np.savez_compressed(os.path.join(target, f"{name}.npz"),
                        meta=np.array(json.dumps(meta)), **arrays)
    return status, dt


def make_prf_golden():
    """PRF streams via the reference's Prg (prg.py:39-65), including the
    reference's own KAT (tests/test_prg_transport.py:14-23) and draws that
    start mid-block."""
    from ring3pc.prg import Prg, derive_pair_seeds, derive_salt
    rng = np.random.default_rng(2024)
    arrays, meta = {}, {"streams": []}
    specs = [(bytes(range(16)), "testvec", [2, 1, 3, 8, 17, 64])]
    for i in range(5):
        seed = rng.integers(0, 256, 16, dtype=np.uint8).tobytes()
        specs.append((seed, f"dom{i}.sha" if i % 2 else "sha", [1, 5, 2, 33, 128, 7]))
    for k, (seed, dom, draws) in enumerate(specs):
        p = Prg(seed, dom)
        outs = [p.draw_u64(n) for n in draws]
        arrays[f"s{k}"] = np.concatenate(outs)
        meta["streams"].append({"seed": seed.hex(), "domain": dom, "draws": draws})
    # draw_bits / draw_base width masks
    p = Prg(bytes(range(16)), "m")
    arrays["bits"] = p.draw_bits(100)
    arrays["base4"] = p.draw_base(64, 4)
    # BLAKE2b pair seeds / salt for a few session seeds
    meta["pair_seeds"] = {}
    for s in (0, 3, 11, 424242):
        master = s.to_bytes(16, "little")
        meta["pair_seeds"][str(s)] = {k: v.hex() for k, v in derive_pair_seeds(master).items()}
        meta["pair_seeds"][str(s)]["salt"] = derive_salt(master).hex()
    np.savez_compressed(os.path.join(HERE, "prf.npz"), meta=np.array(json.dumps(meta)), **arrays)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    ap.add_argument("--scale", action="store_true",
                    help="only the config-scale cases (programs.SCALE_CASES), hashed fixtures")
    a = ap.parse_args()
    if a.scale:
        for name, prog, args, kwargs, sess_kw in programs.SCALE_CASES:
            if a.only and a.only != name:
                continue
            st, dt = run_case(name, prog, args, kwargs, sess_kw, hashed=True)
            print(f"{name:28s} {st:10s} {dt:7.2f}s", flush=True)
        return
    make_prf_golden()
    for name, prog, args, kwargs, sess_kw in programs.CASES:
        if a.only and a.only != name:
            continue
        st, dt = run_case(name, prog, args, kwargs, sess_kw)
        print(f"{name:28s} {st:10s} {dt:7.2f}s")
    for name, prog, args, inj, sess_kw in programs.TAMPER_CASES:
        if a.only and a.only != name:
            continue
        st, dt = run_case(name, prog, args, {}, sess_kw, injection=inj)
        print(f"{name:28s} {st:10s} {dt:7.2f}s")


if __name__ == "__main__":
    main()
