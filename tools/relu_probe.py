"""Secure-ReLU session timing with and without verification (debug aid).

    python tools/relu_probe.py N
"""
import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2411_09287_b200 import nonlinear, verify, host
from paper_2411_09287_b200.runtime import Session
from paper_2411_09287_b200.sharing import Ring, rec, shc_input_mask, shc_input_online
from paper_2411_09287_b200.transport import Phase
from paper_2411_09287_b200 import _lib
N = int(sys.argv[1]); d = 16
rng = np.random.default_rng(1)
xv = np.trunc(rng.normal(0, 4, N) * 2**16).astype(np.int64).astype(np.uint64)
def prog(party, verify_it):
    ring = Ring(64)
    party.enter_phase(Phase.PRE)
    xm = shc_input_mask(party, 0, N, ring)
    mat = nonlinear.relu_prepare(party, xm, N, ring)
    verify.prepare_verification(party, d=d)
    party.round_barrier()
    party.enter_phase(Phase.ONLINE)
    x = shc_input_online(party, 0, xv if party.role == 0 else None, xm, N, ring, "x")
    out = nonlinear.relu_online(party, x, mat)
    party.round_barrier()
    party.enter_phase(Phase.POST)
    v = verify.verify_session(party, d=d, R="auto") if verify_it else (party.freeze_logs() or {})
    return v, rec(party, out, "relu")
for vf in (False, True):
    Session(seed=1).run(prog, vf)
    torch.cuda.synchronize()
    l0 = _lib.load().r3_launch_count()
    t = time.perf_counter()
    res = Session(seed=2).run(prog, vf)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    got = host(res[0][1]); want = np.where(xv.astype(np.int64) >= 0, xv, 0).astype(np.uint64)
    print("verify" if vf else "exec", N, f"{dt*1e3:.1f} ms", f"{N/dt:.3g} relu/s", "ok" if np.array_equal(got, want) else "MISMATCH", res[0][0], "launches", _lib.load().r3_launch_count()-l0, "mem GB", torch.cuda.max_memory_allocated()/1e9)
