"""Host cost of the protocol driver's per-level steps (all three parties,
coop engine): own time of each wrapped function = wall time inside it
minus the time its thread spent parked in the scheduler (other parties'
turns), summed over parties, plus call counts.  Diagnostic only.

    python tools/level_cost.py mulv 20
"""

import collections
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_09287_b200 import _lib, gates, grvec, nonlinear, runtime, sharing, verify  # noqa: E402
from paper_2411_09287_b200.runtime import Session  # noqa: E402

tl = threading.local()
own = collections.Counter()
cnt = collections.Counter()


def parked() -> float:
    return getattr(tl, "parked", 0.0)


def wrap(mod, name, label=None):
    fn = getattr(mod, name)
    label = label or f"{mod.__name__.split('.')[-1]}.{name}"

    def inner(*a, **k):
        t0, p0 = time.perf_counter(), parked()
        try:
            return fn(*a, **k)
        finally:
            own[label] += (time.perf_counter() - t0) - (parked() - p0)
            cnt[label] += 1
    setattr(mod, name, inner)
    return inner


def main():
    kind, lg = sys.argv[1], int(sys.argv[2])
    N = 1 << lg
    if kind.startswith("relu"):
        xh = torch.from_numpy(np.trunc(np.random.default_rng(1).normal(0, 4, N) * 2 ** 16).astype(np.int64)).pin_memory()
        prog = bench.make_relu_program(N, 16)
        args = (xh, kind != "relu_x")          # relu_x: execution only (PRE + ONLINE)
    else:
        prog, _ = bench.make_programs(N, 64, verify.pick_r(N, 64, 64))
        args = ()
    for i in range(3):
        Session(seed=i).run(prog, *args)
    torch.cuda.synchronize()
    orig_yield = runtime._Baton.yield_to_scheduler

    def y(self, ready=None):
        t0 = time.perf_counter()
        try:
            return orig_yield(self, ready)
        finally:
            tl.parked = parked() + time.perf_counter() - t0
    runtime._Baton.yield_to_scheduler = y
    for mod, names in ((verify, ["_gr_dot_folded", "_open_challenge", "_recombine", "_quad", "_level_folds_fused",
                                 "_level_line_evals", "reduce_dimension", "check_inner_product", "_dotsum_terms",
                                 "_round_joint", "_rdim_compute", "_folds16_all", "_reduction_round",
                                 "verify_session", "batch_verify_muls", "batch_verify_dots", "_compress_reduce_first",
                                 "_reduce_second_from_base", "_verify_muls_gf2", "_verify_tail", "prepare_verification",
                                 "_base_fold", "_powers", "_l2_tables", "_reduce_from_base", "_powers_b",
                                 "_base_fold_b", "_block_fold_weights", "_base_tables", "_open_challenge"]),
                       (nonlinear, ["relu_prepare", "relu_online", "edabits_prepare", "dabit_prepare", "_xor_arith",
                                    "a2b", "_ripple_msb_fused", "b2a", "_bit_share", "drelu_online"]),
                       (gates, ["dot_prepare", "mul_prepare", "mul_finish"]),
                       (sharing, ["shc_input_mask", "shc_input_online", "rec"]),
                       (runtime.Party, ["send", "recv", "send_digest", "check_digest", "round_barrier"]),
                       (runtime.Session, ["joint", "defer_check"]),
                       (gates, ["prepare_gate", "dot_finish"]),
                       (sharing, ["sha_random", "sha_input"]),
                       (_lib, ["call", "empty", "zeros"]),
                       (grvec, ["ew", "ew_fields", "gr_lincomb"])):
        for n in names:
            wrap(mod, n)
    # rebind names imported by value
    for mod in (verify, gates, sharing, grvec):
        for n in ("call", "empty", "zeros"):
            if hasattr(mod, n):
                setattr(mod, n, getattr(_lib, n))
    verify.rec = sharing.rec
    reps = 5
    t0 = time.perf_counter()
    for i in range(reps):
        Session(seed=100 + i).run(prog, *args)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / reps
    print(f"{kind} 2^{lg}: {1e3 * wall:.1f} ms per session (instrumented)")
    for k, v in own.most_common(45):
        print(f"  {1e3 * v / reps:8.2f} ms  {cnt[k] / reps:7.0f} calls  {1e6 * v / max(1, cnt[k]):6.1f} us/call  {k}")


if __name__ == "__main__":
    main()
