"""Party programs shared by the golden dumper and the parity tests.

Every program is written once against the reference-shaped public API and
built for a given package (`ring3pc` for the read-only reference when the
golden vectors are generated in the build container, or
`paper_2411_09287_b200` for the B200 implementation under test).  The
structure of each program follows a named program of the reference's own
suite, cited per function; nothing here depends on the package's kernels.
"""

from __future__ import annotations

import importlib
from types import SimpleNamespace

import numpy as np


def build(pkg_name: str) -> SimpleNamespace:
    gates = importlib.import_module(f"{pkg_name}.gates")
    verify = importlib.import_module(f"{pkg_name}.verify")
    sharing = importlib.import_module(f"{pkg_name}.sharing")
    transport = importlib.import_module(f"{pkg_name}.transport")
    nonlinear = importlib.import_module(f"{pkg_name}.nonlinear")
    ppml = importlib.import_module(f"{pkg_name}.ppml")
    circuit = importlib.import_module(f"{pkg_name}.circuit")
    Ring, MVal = sharing.Ring, sharing.MVal
    Phase = transport.Phase
    shc_random, shc_input, rec = sharing.shc_random, sharing.shc_input, sharing.rec
    shc_input_mask, shc_input_online = sharing.shc_input_mask, sharing.shc_input_online

    def mulv(party, lanes, d, R, ell=64, dots_n=0, auto=False):
        """tests/test_verify.py:17-42 (and test_acceptance.py:124-136)."""
        ring = Ring(ell)
        party.enter_phase(Phase.PRE)
        x = shc_random(party, lanes, ring)
        y = shc_random(party, lanes, ring)
        g = gates.mul_prepare(party, x.mask, y.mask, lanes)
        dg = None
        if dots_n:
            xs = shc_random(party, dots_n * 2, ring)
            ys = shc_random(party, dots_n * 2, ring)
            resh = lambda v: MVal(v.mask._map(lambda a: a.reshape(dots_n, 2)),
                                  None if v.m is None else v.m.reshape(dots_n, 2))
            dg = (gates.dot_prepare(party, resh(xs).mask, resh(ys).mask, 2),
                  resh(xs), resh(ys))
        verify.prepare_verification(party, d=d, r_max=max(R, 1) if not auto else 24)
        party.round_barrier()
        party.enter_phase(Phase.ONLINE)
        z = gates.mul_finish(party, g, x, y)
        if dg is not None:
            gates.dot_finish(party, dg[0], dg[1], dg[2])
        party.round_barrier()
        party.enter_phase(Phase.POST)
        if auto:
            out = verify.verify_session(party, d=d, R="auto")
        else:
            out = {"mul": verify.batch_verify_muls(party, ell, d=d, R=R)}
            if dots_n:
                out["dot"] = verify.batch_verify_dots(party, ell, d=d, R=R)
        return {"x": x, "y": y, "z": z, "verdict": out}

    def mul_inputs(party, xv, yv, ell=64):
        """tests/test_gates.py:11-22: owner inputs then one online mul."""
        ring = Ring(ell)
        lanes = len(xv)
        party.enter_phase(Phase.PRE)
        party.enter_phase(Phase.ONLINE)
        x = shc_input(party, 0, np.asarray(xv, dtype=np.uint64)
                      if party.role == 0 else None, lanes, ring, "x")
        y = shc_input(party, 1, np.asarray(yv, dtype=np.uint64)
                      if party.role == 1 else None, lanes, ring, "y")
        z = gates.mul(party, x, y)
        party.round_barrier()
        party.enter_phase(Phase.POST)
        party.freeze_logs()
        return {"z": z, "open": rec(party, z, "z")}

    def bool_mulv(party, lanes, d, R):
        """tests/test_verify.py:122-135 (boolean log, GF(2^d))."""
        ring = Ring(1)
        party.enter_phase(Phase.PRE)
        x = shc_random(party, lanes, ring)
        y = shc_random(party, lanes, ring)
        g = gates.mul_prepare(party, x.mask, y.mask, lanes)
        verify.prepare_verification(party, d=d, r_max=max(R, 1))
        party.round_barrier()
        party.enter_phase(Phase.ONLINE)
        z = gates.mul_finish(party, g, x, y)
        party.round_barrier()
        party.enter_phase(Phase.POST)
        return {"x": x, "y": y, "z": z,
                "verdict": {"mul": verify.batch_verify_muls(party, 1, d=d, R=R)}}

    def trunc(party, xv, t):
        """tests/test_gates.py:167-182 / test_acceptance.py:256-272."""
        ring = Ring(64)
        lanes = len(xv)
        party.enter_phase(Phase.PRE)
        mat = gates.trunc_prepare(party, lanes, t, ring)
        party.enter_phase(Phase.ONLINE)
        x = shc_input(party, 0, np.asarray(xv, dtype=np.uint64)
                      if party.role == 0 else None, lanes, ring, "x")
        one = MVal.public(ring, party.role, np.ones(lanes, dtype=np.uint64))
        g = gates.mul_prepare(party, x.mask, one.mask, lanes, out_mask=mat.rx_mask)
        z = gates.trunc_online(party, gates.mul_finish(party, g, x, one), mat)
        party.round_barrier()
        party.enter_phase(Phase.POST)
        party.freeze_logs()
        zv = rec(party, z, "z")
        out = {"z": z, "open": zv}
        if party.role == 0:
            out["rx_clear"] = mat.rx_clear
            out["rz_clear"] = mat.rz_clear
        return out

    def trunc_verify(party, xv, t, d):
        """Truncation whose two logged bit inner products (gates.py:237-238)
        are then batch-verified (verify.py:294-303) with the multiplication."""
        ring = Ring(64)
        lanes = len(xv)
        party.enter_phase(Phase.PRE)
        mat = gates.trunc_prepare(party, lanes, t, ring)
        verify.prepare_verification(party, d=d)
        party.round_barrier()
        party.enter_phase(Phase.ONLINE)
        x = shc_input(party, 0, np.asarray(xv, dtype=np.uint64)
                      if party.role == 0 else None, lanes, ring, "x")
        one = MVal.public(ring, party.role, np.ones(lanes, dtype=np.uint64))
        g = gates.mul_prepare(party, x.mask, one.mask, lanes, out_mask=mat.rx_mask)
        z = gates.trunc_online(party, gates.mul_finish(party, g, x, one), mat)
        party.round_barrier()
        party.enter_phase(Phase.POST)
        v = verify.verify_session(party, d=d, R="auto")
        return {"z": z, "verdict": v, "open": rec(party, z, "z")}

    def dotv(party, n, lanes, d, R):
        """Batched inner products + Pi_bsv (test_verify.py:17-42 dot branch)."""
        ring = Ring(64)
        party.enter_phase(Phase.PRE)
        xs = shc_random(party, n * lanes, ring)
        ys = shc_random(party, n * lanes, ring)
        resh = lambda v: MVal(v.mask._map(lambda a: a.reshape(n, lanes)),
                              None if v.m is None else v.m.reshape(n, lanes))
        xs, ys = resh(xs), resh(ys)
        g = gates.dot_prepare(party, xs.mask, ys.mask, lanes)
        verify.prepare_verification(party, d=d, r_max=max(R, 1))
        party.round_barrier()
        party.enter_phase(Phase.ONLINE)
        z = gates.dot_finish(party, g, xs, ys)
        party.round_barrier()
        party.enter_phase(Phase.POST)
        v = verify.batch_verify_dots(party, 64, d=d, R=R)
        return {"z": z, "verdict": {"dot": v}}

    def relu(party, xv, d=16, R="auto"):
        """owner-P0 input, relu_prepare, relu_online,
        verify_session (nonlinear.py:295-319; verify.py:321-338)."""
        ring = Ring(64)
        lanes = len(xv)
        party.enter_phase(Phase.PRE)
        xmask = shc_input_mask(party, 0, lanes, ring)
        mat = nonlinear.relu_prepare(party, xmask, lanes, ring)
        verify.prepare_verification(party, d=d)
        party.round_barrier()
        party.enter_phase(Phase.ONLINE)
        x = shc_input_online(party, 0, np.asarray(xv, dtype=np.uint64)
                             if party.role == 0 else None, xmask, lanes, ring, "x")
        out = nonlinear.relu_online(party, x, mat)
        party.round_barrier()
        party.enter_phase(Phase.POST)
        verdict = verify.verify_session(party, d=d, R=R)
        return {"relu": out, "verdict": verdict, "open": rec(party, out, "relu")}

    def a2b_roundtrip(party, xs, ell):
        """tests/test_acceptance.py:294-316."""
        ring = Ring(ell)
        lanes = len(xs)
        party.enter_phase(Phase.PRE)
        eda = nonlinear.edabits_prepare(party, lanes, ring)
        dabs = [nonlinear.dabit_prepare(party, lanes, ring) for _ in range(ell)]
        party.round_barrier()
        party.enter_phase(Phase.ONLINE)
        x = shc_input(party, 0, np.array(xs, dtype=np.uint64)
                      if party.role == 0 else None, lanes, ring, "x")
        bits = nonlinear.a2b(party, x, eda)
        acc = None
        for i in range(ell):
            ai = nonlinear.b2a(party, bits.take(i), dabs[i], ring)
            ai = ai.scale_pub(np.uint64((1 << i) & ring.mask))
            acc = ai if acc is None else acc + ai
        party.round_barrier()
        party.enter_phase(Phase.POST)
        party.freeze_logs()
        return {"open": rec(party, acc, "x2"), "ea": rec(party, eda.arith, "ea")}

    def matmul(party, Xv, Wv, t=16, check=False, d=16):
        """Share matmul + truncation as ppml.infer runs an FC layer
        (ppml.py:304-309, 320-328, 373-381, 412-427): X (M,K) owned by P2,
        W (K,N) owned by P1, gathered (K, M*N) operands, one Pi_dot with the
        truncation input mask as its output mask, then trunc_online."""
        ring = Ring(64)
        M, K = Xv.shape
        N = Wv.shape[1]
        lanes = M * N
        party.enter_phase(Phase.PRE)
        xmask = shc_input_mask(party, 2, M * K, ring)
        wmask = shc_input_mask(party, 1, K * N, ring)
        tr = gates.trunc_prepare(party, lanes, t, ring)
        xi = (np.arange(M)[None, :, None] * K + np.arange(K)[:, None, None]
              + np.zeros((1, 1, N), dtype=np.int64)).reshape(K, lanes)
        wi = (np.arange(K)[:, None, None] * N + np.arange(N)[None, None, :]
              + np.zeros((1, M, 1), dtype=np.int64)).reshape(K, lanes)
        gx = lambda a: a[xi]
        gw = lambda a: a[wi]
        g = gates.dot_prepare(party, xmask._map(gx), wmask._map(gw), lanes,
                              out_mask=tr.rx_mask)
        if check:
            verify.prepare_verification(party, d=d)
        party.round_barrier()
        party.enter_phase(Phase.ONLINE)
        X = shc_input_online(party, 2, Xv.reshape(-1) if party.role == 2 else None,
                             xmask, M * K, ring, "X")
        W = shc_input_online(party, 1, Wv.reshape(-1) if party.role == 1 else None,
                             wmask, K * N, ring, "W")
        gxv = lambda v: MVal(v.mask._map(gx), None if v.m is None else gx(v.m))
        gwv = lambda v: MVal(v.mask._map(gw), None if v.m is None else gw(v.m))
        prod = gates.dot_finish(party, g, gxv(X), gwv(W))
        party.round_barrier()
        z = gates.trunc_online(party, prod, tr)
        party.enter_phase(Phase.POST)
        if check:
            # ppml.py:440-445: verify every log before anything is opened
            return {"verdict": verify.verify_session(party, d=d, R="auto"), "z": z,
                    "open": rec(party, z, "z")}
        party.freeze_logs()
        return {"z": z, "open": rec(party, z, "z")}

    def matmul_gemm(party, Xv, Wv, t=16, check=False, d=16):
        """The matmul program through the GEMM-form gate API
        (paper_2411_09287_b200 only: gates.matmul_prepare / matmul_finish);
        must reproduce the gathered-dot golden run exactly."""
        ring = Ring(64)
        M, K = Xv.shape
        N = Wv.shape[1]
        party.enter_phase(Phase.PRE)
        xmask = shc_input_mask(party, 2, M * K, ring)
        wmask = shc_input_mask(party, 1, K * N, ring)
        tr = gates.trunc_prepare(party, M * N, t, ring)
        g = gates.matmul_prepare(party, xmask, wmask, M, K, N, out_mask=tr.rx_mask)
        if check:
            verify.prepare_verification(party, d=d)
        party.round_barrier()
        party.enter_phase(Phase.ONLINE)
        X = shc_input_online(party, 2, Xv.reshape(-1) if party.role == 2 else None,
                             xmask, M * K, ring, "X")
        W = shc_input_online(party, 1, Wv.reshape(-1) if party.role == 1 else None,
                             wmask, K * N, ring, "W")
        prod = gates.matmul_finish(party, g, X, W)
        party.round_barrier()
        z = gates.trunc_online(party, prod, tr)
        party.enter_phase(Phase.POST)
        if check:
            return {"verdict": verify.verify_session(party, d=d, R="auto"), "z": z,
                    "open": rec(party, z, "z")}
        party.freeze_logs()
        return {"z": z, "open": rec(party, z, "z")}


    def _model(name):
        if name == "snn":
            return ppml.snn_model(np.random.default_rng(0))
        if name == "mlp_tiny":
            m = ppml.ModelSpec((1, 4, 4), [ppml.Layer("fc", dict(din=16, dout=8)), ppml.Layer("relu"),
                                           ppml.Layer("fc", dict(din=8, dout=4)), ppml.Layer("relu"),
                                           ppml.Layer("fc", dict(din=4, dout=3))])
            rng = np.random.default_rng(1)
            m.weights = [rng.normal(0, 0.3, 128), rng.normal(0, 0.4, 32), rng.normal(0, 0.5, 12)]
            return m
        if name == "conv_tiny":
            m = ppml.ModelSpec((1, 6, 6), [
                ppml.Layer("conv", dict(out=2, kh=3, kw=3, sh=1, sw=1, pad=1)), ppml.Layer("relu"),
                ppml.Layer("maxpool", dict(win=2)), ppml.Layer("fc", dict(din=18, dout=3))])
            rng = np.random.default_rng(2)
            m.weights = [rng.normal(0, 0.3, 18), rng.normal(0, 0.3, 54)]
            return m
        raise ValueError(name)

    def _images(model, batch, seed):
        n_in = int(np.prod(model.input_shape))
        return np.random.default_rng(seed).normal(0, 1, (batch, n_in))

    def infer1(party, model_name, img_seed, d=16, check=True):
        """ppml.infer on one image (ppml.py:291-409), the reference's own API."""
        model = _model(model_name)
        img = _images(model, 1, img_seed)[0]
        cfg = ppml.InferConfig(d=d, check=check)
        scores, verdicts = ppml.infer(party, model, img, cfg)
        return {"scores": scores, "verdicts": verdicts}

    def _batched_idx(lay, shape, B):
        """(K, lanes) gather indices of a batched layer (image-major lanes;
        conv lanes (b, oc, p) as the reference orders one image's)."""
        n_img = int(np.prod(shape))
        if lay.kind == "fc":
            din, dout = lay.params["din"], lay.params["dout"]
            b, o = np.meshgrid(np.arange(B), np.arange(dout), indexing="ij")
            i = np.arange(din)[:, None]
            return b.reshape(1, -1) * din + i, o.reshape(1, -1) * din + i
        idx = ppml.conv_indices(shape, lay.params)
        K, P = idx.shape
        out = lay.params["out"]
        b, oc, p = np.meshgrid(np.arange(B), np.arange(out), np.arange(P), indexing="ij")
        b, oc, p = b.reshape(-1), oc.reshape(-1), p.reshape(-1)
        raw = idx[:, p]
        xi = np.where(raw == n_img, B * n_img, b[None, :] * n_img + raw)
        wi = oc[None, :] * K + np.arange(K)[:, None]
        return xi, wi

    def _gmask(m, idx):
        return m._map(lambda a: np.concatenate([np.asarray(a), np.zeros(1, np.uint64)])[idx])

    def infer_batch_gathered(party, model_name, img_seed, batch, d=16, check=True):
        """BASELINE configs 4-5 in the reference's own primitives: ppml.infer
        (ppml.py:291-409) with every per-image lane count scaled by the batch,
        each linear layer one gathered Pi_dot (ppml.py:412-427)."""
        model = _model(model_name)
        imgs = _images(model, batch, img_seed)
        cfg = ppml.InferConfig(d=d, check=check)
        ring = Ring(party.ell)
        shapes = model.shapes()
        B = batch
        party.enter_phase(Phase.PRE)
        n_in = int(np.prod(model.input_shape))
        img_mask = shc_input_mask(party, cfg.data_owner, B * n_in, ring)
        w_masks = [shc_input_mask(party, cfg.model_owner, model.weight_count(l), ring)
                   if model.weight_count(l) else None for l in model.layers]
        plans, cur_mask, cur_shape = [], img_mask, model.input_shape
        for li, lay in enumerate(model.layers):
            lanes = B * int(np.prod(shapes[li]))
            if lay.kind in ("conv", "fc"):
                tr = gates.trunc_prepare(party, lanes, cfg.k, ring)
                xi, wi = _batched_idx(lay, cur_shape, B)
                gate = None
                if cur_mask is not None:
                    gate = gates.dot_prepare(party, _gmask(cur_mask, xi), _gmask(w_masks[li], wi), lanes,
                                             out_mask=tr.rx_mask)
                plans.append(("dot", tr, gate, (xi, wi)))
                cur_mask = tr.rz_mask
            elif lay.kind == "relu":
                mat = nonlinear.relu_prepare(party, cur_mask, lanes, ring) if cur_mask is not None else None
                plans.append(("relu", mat, None, None))
                cur_mask = None
            else:
                plans.append(("maxpool", None, None, None))
                cur_mask = None
            cur_shape = shapes[li]
        if check:
            verify.prepare_verification(party, d=d)
        party.round_barrier()
        party.enter_phase(Phase.ONLINE)
        vals = ppml.encode(imgs.reshape(-1), cfg.k, ring.ell) if party.role == cfg.data_owner else None
        cur = shc_input_online(party, cfg.data_owner, vals, img_mask, B * n_in, ring, "image")
        weights, nw = [], 0
        for li, lay in enumerate(model.layers):
            n = model.weight_count(lay)
            if not n:
                weights.append(None)
                continue
            wv = ppml.encode(model.weights[nw], cfg.k, ring.ell) if party.role == cfg.model_owner else None
            nw += 1
            weights.append(shc_input_online(party, cfg.model_owner, wv, w_masks[li], n, ring, f"w{li}"))
        party.round_barrier()
        cur_shape = model.input_shape
        for li, lay in enumerate(model.layers):
            lanes = B * int(np.prod(shapes[li]))
            kind, mat, gate, ix = plans[li]
            if kind == "dot":
                xi, wi = ix
                gv = lambda v, idx: MVal(_gmask(v.mask, idx), None if v.m is None else
                                         np.concatenate([np.asarray(v.m), np.zeros(1, np.uint64)])[idx])
                xs, ws = gv(cur, xi), gv(weights[li], wi)
                if gate is None:
                    gate = gates.dot_prepare(party, xs.mask, ws.mask, lanes, out_mask=mat.rx_mask)
                prod = gates.dot_finish(party, gate, xs, ws)
                party.round_barrier()
                cur = gates.trunc_online(party, prod, mat)
            elif kind == "relu":
                if mat is None:
                    mat = nonlinear.relu_prepare(party, cur.mask, lanes, ring)
                cur = nonlinear.relu_online(party, cur, mat)
                party.round_barrier()
            else:
                base = ppml._pool_indices(cur_shape, lay.params["win"])
                n_img = int(np.prod(cur_shape))
                idx = (np.arange(B)[None, :, None] * n_img + base[:, None, :]).reshape(base.shape[0], -1)
                cur = nonlinear.maxpool_online(party, ppml._gather(cur, idx), ring)
                party.round_barrier()
            cur_shape = shapes[li]
        party.enter_phase(Phase.POST)
        verdicts = {}
        if check:
            verdicts = verify.verify_session(party, d=d, R="auto")
            if not all(verdicts.values()):
                party.abort(f"verification failed before output reveal: {verdicts}")
        else:
            party.freeze_logs()
        return {"scores": rec(party, cur, "scores"), "verdicts": verdicts}

    def infer_batch(party, model_name, img_seed, batch, d=16, check=True):
        """paper_2411_09287_b200 only: ppml.infer_batch (GEMM-form layers);
        must reproduce infer_batch_gathered's golden run exactly."""
        model = _model(model_name)
        imgs = _images(model, batch, img_seed)
        scores, verdicts = ppml.infer_batch(party, model, imgs, ppml.InferConfig(d=d, check=check))
        return {"scores": scores, "verdicts": verdicts}

    def circ(party, name, d=16, R=1, check=True):
        """tests/test_circuit.py:41-110: circuit.evaluate over a named text
        circuit (CIRCUITS below) with its plaintext inputs."""
        text, values = CIRCUITS[name]
        outs, verdicts = circuit.evaluate(party, circuit.parse(text), values, d, R, check)
        return {"outputs": np.array(outs, dtype=np.uint64), "verdicts": verdicts}

    return SimpleNamespace(circ=circ, matmul_gemm=matmul_gemm, mulv=mulv, mul_inputs=mul_inputs, bool_mulv=bool_mulv,
                           trunc=trunc, trunc_verify=trunc_verify, dotv=dotv, relu=relu,
                           a2b_roundtrip=a2b_roundtrip, matmul=matmul, infer1=infer1,
                           infer_batch_gathered=infer_batch_gathered, infer_batch=infer_batch)


# ---------------------------------------------------------------------------
# Golden case table: (name, program, args, kwargs, session kwargs)
# ---------------------------------------------------------------------------

def _trunc_inputs(n, seed):
    rng = np.random.default_rng(seed)
    xs = rng.integers(-(2 ** 40) + 1, 2 ** 40, n)
    return np.array([int(v) % 2 ** 64 for v in xs], dtype=np.uint64)


def _relu_inputs(n, seed):
    rng = np.random.default_rng(seed)
    vals = np.trunc(rng.normal(0, 4, n) * 2 ** 16).astype(np.int64)
    return vals.astype(np.uint64)


def _mat_inputs(M, K, N, seed):
    rng = np.random.default_rng(seed)
    X = np.trunc(rng.normal(0, 1, (M, K)) * 2 ** 16).astype(np.int64).astype(np.uint64)
    W = np.trunc(rng.normal(0, 1 / 8, (K, N)) * 2 ** 16).astype(np.int64).astype(np.uint64)
    return X, W


def _fx(v, k=8):
    return int(v * 2 ** k) % 2 ** 64


def random_circuit(seed: int, n_gates: int = 14, k: int = 8):
    """Seeded random circuit over every gate kind: products feed TRUNC, and
    RELU / MAXPOOL outputs feed later products, so those products get their
    masks online.  Linear gates only read wires whose mask is known offline
    (the reference's offline pass cannot propagate an online-only mask
    through ADD / SUB / SCALE, circuit.py:176-184), and stacked operand
    lists start with a truncation output when they hold one (the
    reference stacks the first mask's fields, nonlinear.py:248-259, and a
    truncation output's P0 view is sum-only)."""
    rng = np.random.default_rng(seed)
    lines, values, wires, wid = [], {}, [], 0
    online_mask = set()                       # wires whose mask is set online
    truncs = set()                            # sum-only P0 view: truncation lineage
    sparse_first = lambda ids: sorted(ids, key=lambda w: w not in truncs)
    for _ in range(3):
        lines.append(f"INPUT {wid} {int(rng.integers(0, 3))}")
        values[wid] = _fx(float(rng.normal(0, 2)), k)
        wires.append(wid)
        wid += 1
    lines.append(f"CONST {wid} {_fx(0.5, k)}")
    wires.append(wid)
    wid += 1
    for _ in range(n_gates):
        op = str(rng.choice(["ADD", "SUB", "MULT", "DOTT", "SCALE", "RELU", "MAXPOOL"]))
        pick = lambda n: [int(x) for x in rng.choice(wires, size=n)]
        offline = [w for w in wires if w not in online_mask]
        pick_off = lambda n: [int(x) for x in rng.choice(offline, size=n)]
        if op in ("ADD", "SUB"):
            a, b = pick_off(2)
            lines.append(f"{op} {wid} {a} {b}")
            if a in truncs or b in truncs:
                truncs.add(wid)
        elif op == "SCALE":
            a = pick_off(1)[0]
            lines.append(f"SCALE {wid} {int(rng.integers(-3, 4)) % 2 ** 64} {a}")
            if a in truncs:
                truncs.add(wid)
        elif op == "RELU":
            a = pick(1)[0]
            lines.append(f"RELU {wid} {a}")
            online_mask.add(wid)
            if a in truncs:
                truncs.add(wid)
        elif op == "MAXPOOL":
            n = int(rng.integers(2, 5))
            ids = sparse_first(pick(n))
            lines.append(f"MAXPOOL {wid} {n} " + " ".join(map(str, ids)))
            online_mask.add(wid)
            if ids[0] in truncs:
                truncs.add(wid)
        else:                                   # product then truncation
            if op == "MULT":
                a, b = pick(2)
                lines.append(f"MUL {wid} {a} {b}")
            else:
                n = int(rng.integers(1, 4))
                ids = sparse_first(pick(n)) + sparse_first(pick(n))
                lines.append(f"DOT {wid} {n} " + " ".join(map(str, ids)))
            wid += 1
            lines.append(f"TRUNC {wid} {wid - 1} {k}")
            truncs.add(wid)
        wires.append(wid)
        wid += 1
    for w in sorted({wires[-1]} | {int(x) for x in rng.choice(wires[4:], size=3)}):
        lines.append(f"OUTPUT {w}")
    return "\n".join(lines), values


CIRCUITS = {
    # tests/test_circuit.py:41-57
    "mixed": ("INPUT 0 0\nINPUT 1 1\nINPUT 2 2\nCONST 3 11\nMUL 4 0 1\nADD 5 4 2\nSUB 6 5 3\n"
              "SCALE 7 3 6\nDOT 8 2 4 5 6 7\nOUTPUT 7\nOUTPUT 8", {0: 3, 1: 5, 2: 9}),
    # tests/test_circuit.py:92-110
    "trunc_relu_pool": ("INPUT 0 0\nINPUT 1 1\nMUL 2 0 1\nTRUNC 3 2 8\nRELU 4 3\n"
                        "MAXPOOL 5 2 3 4\nOUTPUT 4\nOUTPUT 5", {0: _fx(-1.5), 1: _fx(2.0)}),
    # deferred masks: products whose inputs come out of RELU / MAXPOOL
    "deferred": ("INPUT 0 2\nINPUT 1 1\nRELU 2 0\nMUL 3 2 1\nTRUNC 4 3 8\nMAXPOOL 5 3 4 0 1\n"
                 "DOT 6 2 5 2 1 0\nSCALE 7 0xffffffffffffffff 1\nOUTPUT 4\nOUTPUT 6\nOUTPUT 7",
                 {0: _fx(1.25), 1: _fx(-0.75)}),
    "add_only": ("INPUT 0 0\nINPUT 1 1\nADD 2 0 1\nOUTPUT 2", {0: 1, 1: 2}),
    "random_a": random_circuit(101),
    "random_b": random_circuit(202, n_gates=20),
}


CASES = [
    ("mulv_64_d16_R2", "mulv", (64, 16, 2), {}, {"seed": 3}),
    ("mulv_1024_d16_R2", "mulv", (1024, 16, 2), {}, {"seed": 11}),
    ("mulv_1024_d64_R7", "mulv", (1024, 64, 7), {}, {"seed": 11}),
    ("mulv_100_d64_R3", "mulv", (100, 64, 3), {}, {"seed": 5}),
    ("mulv_1_d16_R0", "mulv", (1, 16, 0), {}, {"seed": 6}),
    ("mulv_37_d2_R1_ell4", "mulv", (37, 2, 1), {"ell": 4}, {"seed": 1, "ell": 4}),
    ("mulv_33_d64_R3_dots5", "mulv", (33, 64, 3), {"dots_n": 5}, {"seed": 0}),
    ("mulv_3000_d64_auto", "mulv", (3000, 64, 0), {"auto": True}, {"seed": 21}),
    ("mulv_513_d8_R4", "mulv", (513, 8, 4), {}, {"seed": 8}),
    ("mulv_200_d32_R2", "mulv", (200, 32, 2), {}, {"seed": 9}),
    ("mul_inputs_small", "mul_inputs", ([3, 2 ** 63, 12345], [4, 2, 2 ** 64 - 1]), {}, {"seed": 0}),
    ("bool_mulv_40_d16_R2", "bool_mulv", (40, 16, 2), {}, {"seed": 0, "ell": 1}),
    ("trunc_small", "trunc", ([98304, 0, (-98304) % 2 ** 64, 12345 << 16], 16), {}, {"seed": 3}),
    ("trunc_1000", "trunc", (_trunc_inputs(1000, 6), 16), {}, {"seed": 66}),
    ("trunc_verify_200_d16", "trunc_verify", (_trunc_inputs(200, 12), 16, 16), {}, {"seed": 12}),
    ("dotv_8x16_d16_R2", "dotv", (8, 16, 16, 2), {}, {"seed": 4}),
    ("relu_64", "relu", (_relu_inputs(64, 1),), {}, {"seed": 1}),
    ("a2b_roundtrip_ell8", "a2b_roundtrip", (list(range(16)), 8), {}, {"seed": 0, "ell": 8}),
    ("matmul_8x8x8", "matmul", _mat_inputs(8, 8, 8, 3), {}, {"seed": 3}),
    ("matmul_12x16x10", "matmul", _mat_inputs(12, 16, 10, 4), {}, {"seed": 4}),
    ("infer1_mlp_tiny", "infer1", ("mlp_tiny", 5), {}, {"seed": 5}),
    ("infer1_conv_tiny", "infer1", ("conv_tiny", 6), {}, {"seed": 6}),
    ("infer1_snn_nocheck", "infer1", ("snn", 7), {"check": False}, {"seed": 7}),
    ("infer1_snn", "infer1", ("snn", 10), {}, {"seed": 10}),
    ("infer_batch_mlp_tiny_b3", "infer_batch_gathered", ("mlp_tiny", 8, 3), {}, {"seed": 8}),
    ("infer_batch_conv_tiny_b2", "infer_batch_gathered", ("conv_tiny", 9, 2), {}, {"seed": 9}),
]

CASES += [
    ("circ_mixed", "circ", ("mixed",), {}, {"seed": 31}),
    ("circ_trunc_relu_pool", "circ", ("trunc_relu_pool",), {}, {"seed": 32}),
    ("circ_deferred_d64", "circ", ("deferred",), {"d": 64, "R": "auto"}, {"seed": 33}),
    ("circ_add_only_R0", "circ", ("add_only",), {"R": 0}, {"seed": 34}),
    ("circ_random_a", "circ", ("random_a",), {}, {"seed": 35}),
    ("circ_random_b_nocheck", "circ", ("random_b",), {"check": False}, {"seed": 36}),
    ("circ_mixed_ell32", "circ", ("mixed",), {"R": 2}, {"seed": 37, "ell": 32}),
]

# Tamper cases: (name, program, args, injections[(site, who, delta, gate, lane)])
TAMPER_CASES = [
    ("tamper_gamma", "mulv", (16, 16, 2), ("gamma", 0, 5, 0, 3), {"seed": 1000}),
    ("tamper_z", "mulv", (16, 16, 2), ("z", 1, 7, 0, 9), {"seed": 1001}),
    ("tamper_mz", "mulv", (16, 16, 2), ("mz", 1, 1, 0, 2), {"seed": 1002}),
    ("tamper_z_msb", "mulv", (64, 16, 2), ("z", 2, 1 << 63, 0, 5), {"seed": 1003}),
    ("tamper_mz_rec_abort", "mul_inputs", ([3], [4]), ("mz", 1, 1, 0, None), {"seed": 0}),
    ("tamper_circ_gamma", "circ", ("mixed",), ("gamma", 0, 1, 0, None), {"seed": 38}),
    ("tamper_vfy_gamma", "mulv", (64, 16, 3), ("vfy.dot.gamma", 0, 11, 2, 0), {"seed": 1004}),
]


# Config-scale cases: sizes where every multi-stage kernel
# pipeline wraps (the d = 64 tensor-core base fold runs >= 4 K-steps per CTA,
# the d = 16 joint level folds see >= 2^14 dense rows, the factorised
# Pi_bsv runs six structured levels).  The reference takes tens of seconds
# per case, so their fixtures keep a SHA-256 per array instead of the raw
# words (tests/golden/scale/*.npz, make_golden.py --scale).
SCALE_CASES = [
    ("mulv_65536_d64_auto", "mulv", (65536, 64, 0), {"auto": True}, {"seed": 41}),
    ("relu_4096_d16_auto", "relu", (_relu_inputs(4096, 2),), {}, {"seed": 42}),
    ("mulv_40000_d16_auto", "mulv", (40000, 16, 0), {"auto": True}, {"seed": 43}),
    ("matmul_v_24x64x40", "matmul", _mat_inputs(24, 64, 40, 5), {"check": True}, {"seed": 44}),
]
