"""Time the UNMODIFIED reference (ring3pc, /root/reference, pure Python +
numpy) on this container's host for the configs the CPU oracle port does not
cover (ReLU, MLP, LeNet); output profiles/ref_cpu_timing.json.

Build container only (the reference cannot travel to the GPU box); the GPU
bench quotes these numbers as `reference_cpu_measured` with this provenance.
The reference runs one single-threaded numpy session (its parties are
greenlets under the coop engine, here the thread-backed stand-in).

    python tools/ref_cpu_timing.py
"""

import json
import os
import platform
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(REPO, "oracle", "refshim"))
sys.path.insert(0, "/root/reference/pkg/src")

from ring3pc import nonlinear, ppml, verify  # noqa: E402
from ring3pc.runtime import Session  # noqa: E402
from ring3pc.sharing import Ring, rec, shc_input_mask, shc_input_online  # noqa: E402
from ring3pc.transport import Phase  # noqa: E402


def relu_prog(N, check):
    rng = np.random.default_rng(1)
    xv = np.trunc(rng.normal(0, 4, N) * 2 ** 16).astype(np.int64).astype(np.uint64)

    def prog(party):
        ring = Ring(64)
        party.enter_phase(Phase.PRE)
        xm = shc_input_mask(party, 0, N, ring)
        mat = nonlinear.relu_prepare(party, xm, N, ring)
        if check:
            verify.prepare_verification(party, d=16)
        party.round_barrier()
        party.enter_phase(Phase.ONLINE)
        x = shc_input_online(party, 0, xv if party.role == 0 else None, xm, N, ring, "x")
        out = nonlinear.relu_online(party, x, mat)
        party.round_barrier()
        party.enter_phase(Phase.POST)
        if check:
            assert all(verify.verify_session(party, d=16, R="auto").values())
        else:
            party.freeze_logs()
        return rec(party, out, "relu")
    return prog


def timed(fn):
    t0 = time.perf_counter()
    fn()
    return time.perf_counter() - t0


def main():
    out = {"host": {"cpu": platform.processor() or "x86_64", "cores": os.cpu_count(),
                    "python": platform.python_version(), "numpy": np.__version__},
           "note": "unmodified reference (pkg/src/ring3pc), one session, coop engine via the "
                   "thread-backed greenlet stand-in; single-threaded numpy", "results": {}}
    res = out["results"]
    for N in (1 << 12, 1 << 14):
        dt = timed(lambda: Session(seed=1).run(relu_prog(N, False)))
        res[f"relu_exec_{N}"] = {"seconds": dt, "per_s": N / dt, "unit": "ReLU/s"}
        print("relu exec", N, dt, flush=True)
    N = 1 << 12
    dt = timed(lambda: Session(seed=1).run(relu_prog(N, True)))
    res[f"relu_verified_{N}"] = {"seconds": dt, "per_s": N / dt, "unit": "ReLU/s"}
    print("relu verified", N, dt, flush=True)
    # C4 / C5 single-image inference (the reference API is one image per session)
    mlp = ppml.ModelSpec((1, 28, 28), [ppml.Layer("fc", dict(din=784, dout=128)), ppml.Layer("relu"),
                                       ppml.Layer("fc", dict(din=128, dout=128)), ppml.Layer("relu"),
                                       ppml.Layer("fc", dict(din=128, dout=10))])
    rng = np.random.default_rng(0)
    mlp.weights = [rng.normal(0, 0.05, 784 * 128), rng.normal(0, 0.1, 128 * 128), rng.normal(0, 0.1, 1280)]
    lenet = ppml.lenet_model()
    lenet.input_shape = (1, 28, 28)
    lenet.layers[0].params["pad"] = 2
    lenet.weights = [rng.normal(0, 0.2, lenet.weight_count(l)) for l in lenet.layers if lenet.weight_count(l)]
    img = np.random.default_rng(0).normal(0, 1, 784)
    for name, model, checks in (("mlp", mlp, (False, True)), ("lenet28", lenet, (False,))):
        for check in checks:
            cfg = ppml.InferConfig(check=check)
            dt = timed(lambda: Session(seed=2).run(lambda party: ppml.infer(party, model, img, cfg)))
            key = f"{name}_{'verified' if check else 'exec'}_1"
            res[key] = {"seconds": dt, "per_s": 1 / dt, "unit": "images/s"}
            print(key, dt, flush=True)
    with open(os.path.join(REPO, "profiles", "ref_cpu_timing.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
