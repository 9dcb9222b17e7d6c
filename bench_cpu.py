"""CPU baselines for bench.py: the UNMODIFIED reference timed on this host.

The reference package (`ring3pc`, pure Python + numpy) is installed once,
unmodified, into `baseline/_ref` (`pip install --no-index --no-deps --target
baseline/_ref <copy of /root/reference/pkg>`); that directory is git-ignored
but travels to the GPU box with the gpurun snapshot.  Each workload below is
one of the reference's own programs run through its public API
(`ring3pc.runtime.Session(seed, engine="threads").run(program)`, the stock
engine that needs no greenlet), one independent session per host process on
all cores, so the figure is the host's whole-CPU throughput.  If the
reference is not importable, the mulv workload falls back to the oracle port
(oracle/mpc.py, a numpy restatement; kind "port") and the others report
`unavailable`.

Workload sizes are fixed per workload (one session takes a few to ~20 s
single-threaded here) and stated in `sample`; throughput is units / wall
time of the parallel round.  Only bench.py (its cpu_baseline legs and
`--impl reference`) imports this module.
"""

from __future__ import annotations

import concurrent.futures as cf
import functools
import multiprocessing as mp
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or platform.machine()


def host_info() -> dict:
    import numpy as np
    return {"cpu_model": cpu_model(), "logical_cores": os.cpu_count(),
            "python": platform.python_version(), "numpy": np.__version__}


@functools.lru_cache(maxsize=None)
def reference_status() -> str | None:
    """None if the unmodified reference imports from baseline/_ref, else why not."""
    if not os.path.isdir(os.path.join(REF_DIR, "ring3pc")):
        return "baseline/_ref/ring3pc not installed"
    code = ("import sys; sys.path.insert(0, %r); import ring3pc, ring3pc.runtime; "
            "assert ring3pc.__file__.startswith(%r)" % (REF_DIR, REF_DIR))
    import subprocess
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    return None if r.returncode == 0 else (r.stderr.strip().splitlines() or ["import failed"])[-1]


# ---------------------------------------------------------------------------
# workloads: (unit, units per session, sample text) + the program, built in
# the worker process against the reference package
# ---------------------------------------------------------------------------

WORKLOADS = {
    # name: (size, unit, description)
    "mulv": (1 << 14, "verified mults/s",
             "mulv (tests/test_acceptance.py:124-136): {n} mults, d=64, R=pick_r(lan), ell=64"),
    "relu_exec": (1 << 14, "ReLU/s",
                  "secure ReLU (nonlinear.py:295-319), {n} lanes, owner P0, no verification"),
    "relu_verified": (1 << 10, "ReLU/s",
                      "secure ReLU, {n} lanes + verify_session(d=16, R=auto)"),
    "matmul": (256, "share-matmul MACs/s",
               "share matmul {n}x{n}x{n} + truncation t=16 (ppml FC-layer algebra, gathered Pi_dot, "
               "ppml.py:412-427)"),
    "mlp_exec": (1, "images/s", "SecureML MLP 784-128-128-10, ppml.infer of {n} image, no verification"),
    "mlp_verified": (1, "images/s", "SecureML MLP 784-128-128-10, ppml.infer of {n} image, verified (d=16)"),
    "lenet_exec": (1, "images/s", "LeNet-5 on 28x28 (pad 2), ppml.infer of {n} image, no verification"),
}


def _units(name: str, n: int) -> float:
    return float(n) ** 3 if name == "matmul" else float(n)


def _ref_program(name: str, n: int):
    """The reference program for one session (imports ring3pc from baseline/_ref)."""
    import numpy as np
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    from ring3pc import gates, nonlinear, ppml, verify
    from ring3pc.sharing import Ring, rec, shc_input_mask, shc_input_online, shc_random
    from ring3pc.transport import Phase

    if name == "mulv":
        d = 64
        R = verify.pick_r(n, 64, d)

        def prog(party):
            ring = Ring(64)
            party.enter_phase(Phase.PRE)
            x = shc_random(party, n, ring)
            y = shc_random(party, n, ring)
            g = gates.mul_prepare(party, x.mask, y.mask, n)
            verify.prepare_verification(party, d=d, r_max=max(R, 1))
            party.round_barrier()
            party.enter_phase(Phase.ONLINE)
            gates.mul_finish(party, g, x, y)
            party.round_barrier()
            party.enter_phase(Phase.POST)
            ok = verify.batch_verify_muls(party, 64, d=d, R=R)
            assert ok
            return ok
        return prog

    if name.startswith("relu"):
        check = name == "relu_verified"
        rng = np.random.default_rng(1)
        xv = np.trunc(rng.normal(0, 4, n) * 2 ** 16).astype(np.int64).astype(np.uint64)

        def prog(party):
            ring = Ring(64)
            party.enter_phase(Phase.PRE)
            xm = shc_input_mask(party, 0, n, ring)
            mat = nonlinear.relu_prepare(party, xm, n, ring)
            if check:
                verify.prepare_verification(party, d=16)
            party.round_barrier()
            party.enter_phase(Phase.ONLINE)
            x = shc_input_online(party, 0, xv if party.role == 0 else None, xm, n, ring, "x")
            out = nonlinear.relu_online(party, x, mat)
            party.round_barrier()
            party.enter_phase(Phase.POST)
            if check:
                assert all(verify.verify_session(party, d=16, R="auto").values())
            else:
                party.freeze_logs()
            return rec(party, out, "relu")
        return prog

    if name == "matmul":
        rng = np.random.default_rng(3)
        M = K = N = n
        Xv = np.trunc(rng.normal(0, 1, (M, K)) * 2 ** 16).astype(np.int64).astype(np.uint64)
        Wv = np.trunc(rng.normal(0, 1 / 64, (K, N)) * 2 ** 16).astype(np.int64).astype(np.uint64)
        lanes = M * N
        xi = (np.arange(M)[None, :, None] * K + np.arange(K)[:, None, None]
              + np.zeros((1, 1, N), dtype=np.int64)).reshape(K, lanes)
        wi = (np.arange(K)[:, None, None] * N + np.arange(N)[None, None, :]
              + np.zeros((1, M, 1), dtype=np.int64)).reshape(K, lanes)

        def prog(party):
            from ring3pc.sharing import MVal
            ring = Ring(64)
            party.enter_phase(Phase.PRE)
            xmask = shc_input_mask(party, 2, M * K, ring)
            wmask = shc_input_mask(party, 1, K * N, ring)
            tr = gates.trunc_prepare(party, lanes, 16, ring)
            g = gates.dot_prepare(party, xmask._map(lambda a: a[xi]), wmask._map(lambda a: a[wi]), lanes,
                                  out_mask=tr.rx_mask)
            party.round_barrier()
            party.enter_phase(Phase.ONLINE)
            X = shc_input_online(party, 2, Xv.reshape(-1) if party.role == 2 else None, xmask, M * K, ring, "X")
            W = shc_input_online(party, 1, Wv.reshape(-1) if party.role == 1 else None, wmask, K * N, ring, "W")
            gx = lambda v: MVal(v.mask._map(lambda a: a[xi]), None if v.m is None else v.m[xi])
            gw = lambda v: MVal(v.mask._map(lambda a: a[wi]), None if v.m is None else v.m[wi])
            prod = gates.dot_finish(party, g, gx(X), gw(W))
            party.round_barrier()
            z = gates.trunc_online(party, prod, tr)
            party.enter_phase(Phase.POST)
            party.freeze_logs()
            return rec(party, z, "z")
        return prog

    # ppml inference, one image per session (the reference API is per image)
    rng = np.random.default_rng(0)
    if name.startswith("mlp"):
        model = ppml.ModelSpec((1, 28, 28), [
            ppml.Layer("fc", dict(din=784, dout=128)), ppml.Layer("relu"),
            ppml.Layer("fc", dict(din=128, dout=128)), ppml.Layer("relu"),
            ppml.Layer("fc", dict(din=128, dout=10))])
        model.weights = [rng.normal(0, 0.05, 784 * 128), rng.normal(0, 0.1, 128 * 128),
                         rng.normal(0, 0.1, 1280)]
    else:
        model = ppml.lenet_model()
        model.input_shape = (1, 28, 28)
        model.layers[0].params["pad"] = 2
        model.weights = [rng.normal(0, 0.2, model.weight_count(lay)) for lay in model.layers
                         if model.weight_count(lay)]
    img = np.random.default_rng(0).normal(0, 1, 784)
    cfg = ppml.InferConfig(check=name.endswith("verified"))

    def prog(party):
        return ppml.infer(party, model, img, cfg)
    return prog


def _job(args):
    """One independent reference session in this worker process."""
    name, n, seed, kind = args
    t0 = time.perf_counter()
    if kind == "port":
        sys.path.insert(0, ROOT)
        from oracle import mpc
        from oracle.verify_model import pick_r
        res = mpc.mulv(seed=seed, lanes=n, d=64, R=pick_r(n, 64, 64))
        assert res.verdict
    else:
        prog = _ref_program(name, n)
        from ring3pc.runtime import Session
        Session(seed=seed, engine="threads").run(prog)
    return time.perf_counter() - t0


def pool(procs: int | None = None) -> cf.ProcessPoolExecutor:
    """A warmed-up pool of spawned worker processes (one per core by default)."""
    procs = procs or os.cpu_count() or 1
    ex = cf.ProcessPoolExecutor(max_workers=procs, mp_context=mp.get_context("spawn"))
    list(ex.map(_noop, range(procs)))
    ex.procs = procs
    return ex


def measure(name: str, procs: int | None = None, budget_s: float = 10.0, size: int | None = None,
            seed0: int = 100, max_rounds: int = 64, executor: cf.ProcessPoolExecutor | None = None) -> dict:
    """Whole-host throughput of one workload: `procs` independent reference
    sessions at a time (default: every logical core), rounds repeated until
    `budget_s` of wall time has passed (at least one round)."""
    n0, unit, desc = WORKLOADS[name]
    n = size or n0
    why = reference_status()
    kind = "reference"
    if why is not None:
        if name != "mulv":
            return {"unavailable": why, "unit": unit}
        kind = "port"
    own = executor is None
    ex = pool(procs) if own else executor
    procs = ex.procs
    try:
        t0 = time.perf_counter()
        per = []
        rounds = 0
        while rounds < max_rounds and (rounds == 0 or time.perf_counter() - t0 < budget_s):
            per += list(ex.map(_job, [(name, n, seed0 + rounds * procs + i, kind) for i in range(procs)]))
            rounds += 1
        wall = time.perf_counter() - t0
    finally:
        if own:
            ex.shutdown()
    units = _units(name, n) * procs * rounds
    src = ("unmodified reference ring3pc from baseline/_ref, Session(engine='threads')" if kind == "reference"
           else f"oracle port oracle/mpc.py (reference not importable: {why})")
    return {"value": units / wall, "unit": unit, "cores": procs, "kind": kind,
            "sample": f"{procs} independent sessions x {rounds} round(s), each: {desc.format(n=n)}; "
                      f"{src}; wall {wall:.1f}s, median session {sorted(per)[len(per) // 2]:.2f}s",
            "single_session_s": sorted(per)[len(per) // 2],
            "host": host_info()}


def _noop(_):
    return 0


if __name__ == "__main__":
    import json
    for w in sys.argv[1:] or ["mulv"]:
        print(json.dumps({w: measure(w, procs=int(os.environ.get("PROCS", "0")) or None)}), flush=True)
