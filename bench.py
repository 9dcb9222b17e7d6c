"""Benchmark: verified 3PC multiplications per second on B200.

Workload (BASELINE.json configs[1]): the reference's `mulv` program
(tests/test_acceptance.py:124-136) -- x, y = shc_random over Z_2^64, one
batched Pi_mul, prepare_verification, online mul_finish, then the GR(2^64, d)
batch verification Pi_mulv -- run end to end through the drop-in API
(`Session(seed).run(program)`), all three parties simulated on each GPU.
A "step" is one complete verified session over N multiplications; the
default N = 2^25 per GPU is config 2's sweep end, 2^28, at 8 GPUs (weak
scaling), and the side key `mulv_sweep` covers 2^20 .. 2^26 on one GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--log2n L] [--d D]
                    [--R R|auto] [--impl b200|reference]

One process per GPU (torchrun for N > 1).  Ranks run independent sessions
over N multiplications each (weak scaling; the verification of a batch is a
single inner-product check, shards never need a collective on this path).
Prints one JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import gc
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "verified 3PC mults/sec and secure ReLU comparisons/sec at 1/2/4/8 B200 vs CPU ref"
UNIT = "verified mults/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    # 2^25 multiplications per GPU: config 2's sweep end (2^28) at 8 GPUs,
    # weak scaling (every N runs the same per-GPU batch)
    ap.add_argument("--log2n", type=int, default=25)
    ap.add_argument("--d", type=int, default=64)
    ap.add_argument("--R", default="auto")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--engine", default="coop", choices=["coop", "threads"])
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo only to test the N > 1 path on fewer GPUs than ranks")
    ap.add_argument("--e2e-steps", type=int, default=16)
    ap.add_argument("--cpu-seconds", type=float, default=16.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-step-profile", action="store_true",
                    help="skip the headline's per-kernel table and joint=False session")
    ap.add_argument("--profile-kernel", default="r3_gr_matmul2_tc")
    ap.add_argument("--relu-log2n", type=int, default=16)
    ap.add_argument("--relu-sweep-log2n", type=int, default=20)
    ap.add_argument("--mulv-sweep", default="20,22,24,26,27",
                    help="comma list of log2 batch sizes for the config-2 sweep on one GPU ('' = off)")
    ap.add_argument("--mulv-variants", default="24:16:auto,24:64:7",
                    help="extra config-2 points log2n:d:R (R an integer or auto = pick_r); '' = off")
    ap.add_argument("--matmul-n", type=int, default=4096)
    ap.add_argument("--matmul-verified-rows", type=int, default=512,
                    help="rows of X per verified C3 session (0 = skip the verified C3 leg)")
    ap.add_argument("--mlp-batch", type=int, default=4096)
    ap.add_argument("--mlp-verified-batch", type=int, default=4096)
    ap.add_argument("--lenet-batch", type=int, default=1024)
    ap.add_argument("--lenet-verified-batch", type=int, default=256)
    return ap.parse_args()


# ---------------------------------------------------------------------------
# CPU baselines: the unmodified reference on the host cores (bench_cpu.py)
# ---------------------------------------------------------------------------

def cpu_leg(workload: str, budget_s: float) -> dict:
    """Same-run CPU baseline of one workload (rank 0, N = 1): the reference's
    own program on every host core (bench_cpu.measure)."""
    import bench_cpu
    try:
        return bench_cpu.measure(workload, budget_s=budget_s)
    except Exception as e:  # noqa: BLE001 - a baseline failure must not sink the GPU line
        return {"unavailable": f"{type(e).__name__}: {e}"[:300]}


# ---------------------------------------------------------------------------
# clocks sampling during the timed region
# ---------------------------------------------------------------------------

class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._pump, daemon=True).start()
            # nvidia-smi takes a while to start: the timed region (a fraction
            # of a second) must not begin before the sampler is running
            t0 = time.perf_counter()
            while not self.lines and time.perf_counter() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.01)
            self.lines.clear()
        except OSError:
            self.proc = None
        return self

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            if not self.lines:                 # region shorter than one interval
                time.sleep(0.06)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sms.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sms)}


# ---------------------------------------------------------------------------
# programs
# ---------------------------------------------------------------------------

def make_programs(N: int, d: int, R: int):
    from paper_2411_09287_b200 import gates, verify
    from paper_2411_09287_b200._lib import StagedInput
    from paper_2411_09287_b200.sharing import (Ring, rec, shc_input_mask, shc_input_online,
                                               shc_random)
    from paper_2411_09287_b200.transport import Phase

    def mulv(party):
        """tests/test_acceptance.py:124-136."""
        ring = Ring(64)
        party.enter_phase(Phase.PRE)
        x = shc_random(party, N, ring)
        y = shc_random(party, N, ring)
        g = gates.mul_prepare(party, x.mask, y.mask, N)
        verify.prepare_verification(party, d=d, r_max=max(R, 1))
        party.round_barrier()
        party.enter_phase(Phase.ONLINE)
        gates.mul_finish(party, g, x, y)
        party.round_barrier()
        party.enter_phase(Phase.POST)
        return verify.batch_verify_muls(party, 64, d=d, R=R)

    def e2e(party, xh, yh, pre=None, nxt=None):
        """Owner inputs from pinned host memory (P0: x, P1: y), verified
        product opened and copied back to the host.  pre: input copies of
        this session already started (by the previous session, see nxt);
        nxt(role, host): called by the owners when verification starts, to
        start the NEXT session's input copies on the side copy stream, so
        they overlap this session's verification."""
        ring = Ring(64)
        party.enter_phase(Phase.PRE)
        # owners start their input copies now (side stream), overlapping PRE,
        # unless the previous session already did
        pre = pre or {}
        xs = (pre.get(0) or StagedInput(xh)) if party.role == 0 else None
        ys = (pre.get(1) or StagedInput(yh)) if party.role == 1 else None
        xm = shc_input_mask(party, 0, N, ring)
        ym = shc_input_mask(party, 1, N, ring)
        g = gates.mul_prepare(party, xm, ym, N)
        verify.prepare_verification(party, d=d, r_max=max(R, 1))
        party.round_barrier()
        party.enter_phase(Phase.ONLINE)
        x = shc_input_online(party, 0, xs, xm, N, ring, "x")
        y = shc_input_online(party, 1, ys, ym, N, ring, "y")
        z = gates.mul_finish(party, g, x, y)
        party.round_barrier()
        party.enter_phase(Phase.POST)
        if nxt is not None and party.role in (0, 1):
            nxt(party.role, xh if party.role == 0 else yh)
        if not verify.batch_verify_muls(party, 64, d=d, R=R):
            party.abort("verification failed")
        out = rec(party, z, "z")
        return out if party.role == 0 else None

    return mulv, e2e


def make_relu_program(N: int, d: int = 16):
    """x owned by P0, relu_prepare in PRE, relu_online,
    verify_session(d, R="auto") in POST (nonlinear.py:295-319)."""
    from paper_2411_09287_b200 import nonlinear, verify
    from paper_2411_09287_b200.sharing import Ring, rec, shc_input_mask, shc_input_online
    from paper_2411_09287_b200.transport import Phase

    def relu(party, xh, check):
        ring = Ring(64)
        party.enter_phase(Phase.PRE)
        xm = shc_input_mask(party, 0, N, ring)
        mat = nonlinear.relu_prepare(party, xm, N, ring)
        if check:
            verify.prepare_verification(party, d=d)
        party.round_barrier()
        party.enter_phase(Phase.ONLINE)
        x = shc_input_online(party, 0, xh if party.role == 0 else None, xm, N, ring, "x")
        out = nonlinear.relu_online(party, x, mat)
        party.round_barrier()
        party.enter_phase(Phase.POST)
        if check:
            v = verify.verify_session(party, d=d, R="auto")
            if not all(v.values()):
                party.abort("verification failed")
        else:
            party.freeze_logs()
        return rec(party, out, "relu")

    return relu


def aes_blocks(sess) -> int:
    """AES-128 blocks of keystream the session's protocol consumed: every
    distinct pairwise stream (pair, domain) read up to its final offset
    (both holders read the same words; the GPU generates them once)."""
    seen = {}
    for p in sess.parties:
        for key, st in p._prgs.items():
            seen[key] = max(seen.get(key, 0), st.offset)
    return sum(-(-v // 16) for v in seen.values())


def prf_peak_blocks(torch, lib) -> float:
    """Measured bulk keystream rate of the PRF kernel (r3_prf_ctr, four-table
    AES, 2^27 words = 2^26 blocks): the ceiling an AES-bound step runs
    against (LDS-bound)."""
    import ctypes as C
    from paper_2411_09287_b200 import prg
    rk = prg.round_keys(bytes(range(16)))
    n = 1 << 27
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    lib.call("r3_prf_ctr", rk, 0, n, (1 << 64) - 1, 0, out.data_ptr(), lib.stream())
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(3):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        lib.call("r3_prf_ctr", rk, 0, n, (1 << 64) - 1, 0, out.data_ptr(), lib.stream())
        b.record()
        torch.cuda.synchronize()
        best = max(best, (n // 2) / (a.elapsed_time(b) / 1e3))
    del out
    return best


def relu_rates(N_total: int, d: int, steps: int, rank: int, world: int, prof: bool = True) -> dict:
    """Secure ReLU/s (execution and verified) on C1-shaped inputs: N_total
    lanes (normal(0, 4) fixed point, default_rng(1)) sharded over the ranks;
    each rank runs its shard as one session (x owned by P0, relu_prepare /
    relu_online / verify_session(d, auto) / open), the opened shards are
    all-gathered to rank 0 and compared with max(x, 0) there.  Timing: CUDA
    events around `steps` sessions per rank (host protocol driver included),
    max over ranks."""
    import numpy as np
    import torch
    from paper_2411_09287_b200 import _lib
    from paper_2411_09287_b200 import dist as pdist
    from paper_2411_09287_b200.runtime import Session
    n = N_total // world
    rng = np.random.default_rng(1)
    xv_all = np.trunc(rng.normal(0, 4, N_total) * 2 ** 16).astype(np.int64)
    xh = torch.from_numpy(xv_all[rank * n:(rank + 1) * n].copy()).pin_memory()
    want = np.where(xv_all >= 0, xv_all, 0)
    prog = make_relu_program(n, d)
    out = {"N": N_total, "N_per_gpu": n, "n_gpus": world, "d": d, "R": "auto (pick_r, lan)", "unit": "ReLU/s",
           "timing": f"median of {steps} complete sessions per rank (CUDA events around each, host protocol "
                     f"driver inside the region) after 2 warm-up sessions, max over ranks"}
    for check in (False, True):
        key = "verified" if check else "exec"
        for w in range(2):                      # warm-up (allocator, tables)
            Session(seed=pdist.session_seed(rank, w, stream=10)).run(prog, xh, check)
        gc.collect()
        pdist.barrier()
        torch.cuda.synchronize()
        times = []
        for i in range(steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            sess = Session(seed=pdist.session_seed(rank, 2 + i, stream=10 + check))
            res = sess.run(prog, xh, check)
            b.record()
            b.synchronize()
            times.append(a.elapsed_time(b) / 1e3)
        dt = pdist.max_over_ranks(statistics.median(times))
        full = pdist.gather_outputs(res[0])
        if rank == 0:
            got = full.cpu().numpy()
            assert np.array_equal(got, want), "relu output mismatch"
        out[key] = N_total / dt
        out[key + "_ms"] = dt * 1e3
        if not check:
            out["aes_blocks_per_lane"] = aes_blocks(sess) / n
        if prof and rank == 0:
            # one more session under the per-call profiler (outside the timing)
            cp = CallProfiler()
            _lib.CALL_HOOK = cp.hook
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            Session(seed=pdist.session_seed(rank, 99, stream=10 + check)).run(prog, xh, check)
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            _lib.CALL_HOOK = None
            out[key + "_kernels"] = cp.table(wall)
    out["check"] = "opened ReLU equals max(x, 0) on every lane (gathered on rank 0)"
    return out


def mulv_sweep(sizes, d: int, steps: int = 3, variants=()) -> dict:
    """Config 2's sweep on one GPU: verified mults/s per batch size (same
    program as the headline, R = pick_r), median of `steps` sessions after
    one warm-up, with the peak device memory; a size that does not fit in
    HBM is reported as such (2^28 is meant for 8 GPUs: 2^25 per rank).
    `variants`: extra (log2n, d, R) points -- SURVEY 8(d) C2 also names
    d = 16 and the fixed R = 7 beside d = 64 with pick_r."""
    import torch
    from paper_2411_09287_b200 import _lib, verify
    from paper_2411_09287_b200.runtime import Session
    out = {"unit": UNIT, "d": d, "timing": f"median of {steps} sessions after 1 warm-up, wall clock incl. host",
           "points": []}
    todo = [(lg, d, None) for lg in sizes] + list(variants)
    for lg, dd, r_fixed in todo:
        N = 1 << lg
        R = verify.pick_r(N, 64, dd) if r_fixed is None else r_fixed
        prog, _ = make_programs(N, dd, R)
        torch.cuda.empty_cache()
        torch.cuda.reset_peak_memory_stats()
        point = {"log2n": lg, "d": dd, "R": R, "R_rule": "pick_r(lan)" if r_fixed is None else "fixed"}
        try:
            Session(seed=1).run(prog)
            times = []
            for i in range(steps):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                ok = Session(seed=2 + i).run(prog)
                torch.cuda.synchronize()
                times.append(time.perf_counter() - t0)
            assert all(ok), "honest mulv rejected"
        except (torch.OutOfMemoryError, _lib.KernelError) as e:
            # 2^27 needs about 140 GiB: a point that does not fit is recorded
            if isinstance(e, _lib.KernelError) and "memory" not in str(e).lower():
                raise
            point["fits"] = False
            out["points"].append(point)
            torch.cuda.empty_cache()
            continue
        dt = statistics.median(times)
        point.update({"value": N / dt, "ms": dt * 1e3, "peak_gib": torch.cuda.max_memory_allocated() / 2 ** 30})
        out["points"].append(point)
    torch.cuda.empty_cache()
    return out


def matmul_c3(n: int, steps: int, rank: int, world: int, verified_rows: int = 256) -> dict:
    """BASELINE config C3: share-domain matmul n x n x n over Z_2^64 with
    truncation t = 16 (ppml linear-layer algebra, X owned by P2, W by P1,
    fixed-point encode(normal), default_rng(3)), through
    gates.matmul_prepare/finish + trunc_prepare/trunc_online.  With N > 1
    ranks the rows of X are sharded (each rank n/N x n x n against the whole
    W) and the opened row blocks are all-gathered to rank 0."""
    import numpy as np
    import torch
    from paper_2411_09287_b200 import _lib, gates, verify
    from paper_2411_09287_b200 import dist as pdist
    from paper_2411_09287_b200.runtime import Session
    from paper_2411_09287_b200.sharing import Ring, rec, shc_input_mask, shc_input_online
    from paper_2411_09287_b200.transport import Phase

    M = n // world
    rng = np.random.default_rng(3)
    Xf = rng.normal(0, 1, (n, n))
    Wf = rng.normal(0, 1 / 64, (n, n))
    enc = lambda a: torch.from_numpy(np.ascontiguousarray(np.trunc(a * 2 ** 16).astype(np.int64))).pin_memory()
    Xh, Wh = enc(Xf[rank * M:(rank + 1) * M]), enc(Wf)

    def prog(party, open_out, rows=None, check=False):
        """One session over `rows` (default: all M) rows of this rank's X
        block; check=True logs the GEMM-form dot batch and the truncation's
        bit dots and runs verify_session(d=16, R=auto) before opening
        (ppml.py:440-445; the factorised Pi_bsv of verify.py section 3c)."""
        lo, hi = rows if rows is not None else (0, M)
        m = hi - lo
        ring = Ring(64)
        party.enter_phase(Phase.PRE)
        xm = shc_input_mask(party, 2, m * n, ring)
        wm = shc_input_mask(party, 1, n * n, ring)
        tr = gates.trunc_prepare(party, m * n, 16, ring)
        g = gates.matmul_prepare(party, xm, wm, m, n, n, out_mask=tr.rx_mask)
        if check:
            verify.prepare_verification(party, d=16)
        party.round_barrier()
        party.enter_phase(Phase.ONLINE)
        X = shc_input_online(party, 2, Xh[lo:hi].reshape(-1) if party.role == 2 else None, xm, m * n, ring, "X")
        W = shc_input_online(party, 1, Wh.reshape(-1) if party.role == 1 else None, wm, n * n, ring, "W")
        z = gates.trunc_online(party, gates.matmul_finish(party, g, X, W, log=check), tr)
        party.round_barrier()
        party.enter_phase(Phase.POST)
        if check:
            v = verify.verify_session(party, d=16, R="auto")
            if not all(v.values()):
                party.abort("verification failed")
        else:
            party.freeze_logs()
        return rec(party, z, "z") if open_out else None

    out = Session(seed=pdist.session_seed(rank, 0, stream=20)).run(prog, True)[0]
    full = pdist.gather_outputs(out)
    torch.cuda.synchronize()
    pdist.barrier()
    timer = KernelTimer("r3_u64_gemm_tc")
    _lib.CALL_HOOK = timer.hook
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(steps):
        Session(seed=pdist.session_seed(rank, 1 + i, stream=20)).run(prog, False)
    b.record()
    torch.cuda.synchronize()
    _lib.CALL_HOOK = None
    sec = pdist.max_over_ranks(a.elapsed_time(b) / 1e3 / steps)
    gemm_s = timer.seconds()
    res = {"n": n, "n_gpus": world, "rows_per_gpu": M, "ms_per_matmul": sec * 1e3, "matmuls_per_s": 1 / sec,
           "u64_macs_per_s": n ** 3 / sec,
           "scope": "PRE (masks, trunc_prepare, Gamma) + ONLINE (inputs H2D, GEMM legs, trunc_online), "
                    "one complete session per matmul"}
    vfull = None
    if verified_rows:
        # verified C3: the same n x n x n matmul + truncation with every log
        # verified, as sessions over row blocks of `verified_rows` rows (one
        # session's truncation bit-dot log for all n^2 outputs -- 64 x 2^24
        # logged products -- exceeds HBM in the dense verification levels)
        blocks = [(lo, min(M, lo + verified_rows)) for lo in range(0, M, verified_rows)]
        Session(seed=pdist.session_seed(rank, 0, stream=21)).run(prog, False, blocks[0], True)
        torch.cuda.synchronize()
        pdist.barrier()
        a.record()
        vouts = []
        for i, blk in enumerate(blocks):
            vouts.append(Session(seed=pdist.session_seed(rank, 1 + i, stream=21)).run(prog, True, blk, True)[0])
        b.record()
        torch.cuda.synchronize()
        vsec = pdist.max_over_ranks(a.elapsed_time(b) / 1e3)
        vfull = pdist.gather_outputs(torch.cat([v.reshape(-1) for v in vouts]))
        res["verified"] = {"ms_per_matmul": vsec * 1e3, "matmuls_per_s": 1 / vsec,
                           "sessions_per_gpu": len(blocks), "rows_per_session": verified_rows,
                           "d": 16, "R": "auto", "verdict": "every session accepted (verify_session)",
                           "scope": "per session: PRE, ONLINE, verify_session over the GEMM-form dot batch "
                                    "(factorised Pi_bsv) and the truncation bit dots, open"}
    if rank == 0:
        # probabilistic truncation: |open - X W / 2^16| <= 1 ulp on sampled entries
        Xi = np.trunc(Xf * 2 ** 16).astype(np.int64)
        Wi = np.trunc(Wf * 2 ** 16).astype(np.int64)
        rs = np.random.default_rng(5)
        idx = rs.integers(0, n, (64, 2))
        exact = [sum(int(Xi[r, k]) * int(Wi[k, c]) for k in range(n)) for r, c in idx]
        for what, t in (("exec", full), ("verified", vfull)):
            if t is None:
                continue
            got = t.cpu().numpy().reshape(n, n)
            err = max(abs(int(got[r, c]) - (int(v) >> 16)) for (r, c), v in zip(idx, exact))
            assert err <= 1, f"matmul+trunc ({what}) off by {err}"
        res["check"] = "64 sampled outputs (gathered on rank 0) within 1 ulp of trunc(XW / 2^16), exec and verified"
        cublas8 = int8_peak_ops(torch)
        peak8 = max(cublas8, INT8_DENSE_NOMINAL)
        res["gemm_roofline"] = {
            "bound": "tensor", "kernel": "r3_u64_gemm_tc",
            "achieved": timer.work / gemm_s / 1e12 if gemm_s else None, "peak": peak8 / 1e12,
            "unit": "int8 TOP/s", "frac": timer.work / gemm_s / peak8 if gemm_s else None,
            "launches": timer.launches, "kernel_share_of_step": gemm_s / steps / sec,
            "cublaslt_int8_measured": cublas8 / 1e12,
            "peak_source": "nominal dense int8 of B200 (4.5 POPS; MEASURED_PEAKS.json has no int8 entry and "
                           "the in-run cuBLASLt int8 torch._int_mm 8192^3 figure is below this kernel)",
            "work": "2 x 36 limb MACs x M x N x sum(K) per launch"}
        # whole-step kernel table (one more session under the per-call profiler)
        cp = CallProfiler()
        _lib.CALL_HOOK = cp.hook
        t0 = time.perf_counter()
        sess = Session(seed=pdist.session_seed(rank, 99, stream=20))
        sess.run(prog, False)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        _lib.CALL_HOOK = None
        res["kernels"] = cp.table(wall)
        blocks = aes_blocks(sess)
        res["aes_blocks"] = blocks
        res["aes_roofline"] = {"bound": "aes", "achieved": blocks / sec / 1e9, "unit": "G AES blocks/s",
                               "what": "keystream the session consumes (trunc_prepare bit matrices, masks) "
                                       "over the whole matmul step"}
    return res


def _plain_forward(model, imgs):
    """float64 forward pass of the model (conv via the same patch maps)."""
    import numpy as np
    from paper_2411_09287_b200 import ppml
    outs = []
    for img in imgs:
        cur, shape, wi = img.reshape(-1), model.input_shape, 0
        for lay, out_shape in zip(model.layers, model.shapes()):
            if lay.kind == "fc":
                W = model.weights[wi].reshape(lay.params["dout"], lay.params["din"])
                wi += 1
                cur = W @ cur
            elif lay.kind == "conv":
                idx = ppml.conv_indices(shape, lay.params)
                W = model.weights[wi].reshape(lay.params["out"], -1)
                wi += 1
                cur = (W @ np.concatenate([cur, [0.0]])[idx]).reshape(-1)
            elif lay.kind == "relu":
                cur = np.maximum(cur, 0)
            else:
                idx = ppml._pool_indices(shape, lay.params["win"])
                cur = cur[idx].max(axis=0)
            shape = out_shape
        outs.append(cur)
    return np.array(outs)


def ppml_rates(name: str, batch: int, verified_batch: int, rank: int, world: int,
               verified_total: int = 0) -> dict:
    """BASELINE configs 4 / 5: batched private inference through
    ppml.infer_batch (model owner P1, data owner P2, k = 16, d = 16, R auto),
    synthetic MNIST-shaped images normal(0, 1) from default_rng(0) and
    random-init weights.  Exec = PRE + ONLINE (no
    verification), verified = with verify_session before the scores open.
    With N > 1 ranks the images are sharded (batch / N per rank, one
    session each) and the opened scores all-gathered to rank 0, where they
    are compared with a float forward pass."""
    import numpy as np
    import torch
    from paper_2411_09287_b200 import _lib, ppml
    from paper_2411_09287_b200 import dist as pdist
    from paper_2411_09287_b200.runtime import Session
    model = (ppml.secureml_model if name == "mlp" else ppml.lenet28_model)(np.random.default_rng(0))
    out = {"model": "SecureML MLP 784-128-128-10" if name == "mlp" else "LeNet-5 (28x28, pad 2)",
           "unit": "images/s", "k": 16, "d": 16, "R": "auto", "n_gpus": world}
    n_in = int(np.prod(model.input_shape))
    for check, B in ((False, batch), (True, verified_batch)):
        if not B:
            continue
        b = B // world
        imgs = np.random.default_rng(0).normal(0, 1, (B, n_in))
        mine = imgs[rank * b:(rank + 1) * b]
        cfg = ppml.InferConfig(check=check)
        prog = lambda party: ppml.infer_batch(party, model, mine, cfg)
        Session(seed=pdist.session_seed(rank, 0, stream=30 + check)).run(prog)
        pdist.barrier()
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        res = Session(seed=pdist.session_seed(rank, 1, stream=30 + check)).run(prog)
        e.record()
        torch.cuda.synchronize()
        dt = pdist.max_over_ranks(a.elapsed_time(e) / 1e3)
        if check:
            assert all(res[0][1].values()), "verification rejected"
        full = pdist.gather_outputs(res[0][0])
        key = "verified" if check else "exec"
        if rank == 0:
            scores = ppml.decode(full, 16).reshape(B, -1)
            err = float(np.abs(scores - _plain_forward(model, imgs)).max())
            assert err < 0.05, f"{name} scores off by {err}"
            out[key + "_max_abs_err_vs_float"] = err
            cp = CallProfiler()
            _lib.CALL_HOOK = cp.hook
            t0 = time.perf_counter()
            Session(seed=pdist.session_seed(rank, 99, stream=30 + check)).run(prog)
            torch.cuda.synchronize()
            _lib.CALL_HOOK = None
            out[key + "_kernels"] = cp.table(time.perf_counter() - t0)
        out[key] = B / dt
        out[key + "_batch"] = B
        out[key + "_ms"] = dt * 1e3
    if verified_total > verified_batch > 0:
        # the config batch, verified: sequential sessions of verified_batch
        # images per rank, each a complete PRE / ONLINE / verify / open run
        imgs = np.random.default_rng(1).normal(0, 1, (verified_total, n_in))
        cfg = ppml.InferConfig(check=True)
        per_rank = verified_total // world
        lo_r = rank * per_rank
        outs = []
        pdist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, lo in enumerate(range(lo_r, lo_r + per_rank, verified_batch)):
            part = imgs[lo:min(lo + verified_batch, lo_r + per_rank)]
            res = Session(seed=pdist.session_seed(rank, 100 + i, stream=32)).run(
                lambda party: ppml.infer_batch(party, model, part, cfg))
            assert all(res[0][1].values()), "verification rejected"
            outs.append(res[0][0])
        torch.cuda.synchronize()
        dt = pdist.max_over_ranks(time.perf_counter() - t0)
        full = pdist.gather_outputs(torch.cat(outs))
        if rank == 0:
            sc = ppml.decode(full, 16).reshape(verified_total, -1)
            err = float(np.abs(sc - _plain_forward(model, imgs)).max())
            assert err < 0.05, f"{name} scores off by {err}"
            out["verified_config_batch"] = {"images": verified_total,
                                            "sessions_per_gpu": -(-per_rank // verified_batch),
                                            "images_per_s": verified_total / dt, "ms": dt * 1e3,
                                            "max_abs_err_vs_float": err}
    return out


class KernelTimer:
    """CUDA events around every launch of one library entry point, on the
    launching (current) stream."""

    def __init__(self, name: str):
        self.name = name
        # the batched form of an entry point launches the same kernel
        self.names = {name, name + "_multi"}
        self.events = []
        self.work = 0
        self.launches = 0

    def hook(self, name, args, run):
        import torch
        if name not in self.names:
            return run()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        rc = run()
        b.record()
        self.events.append((a, b))
        self.launches += 1
        self.work += work_of(name, args)
        return rc

    def seconds(self) -> float:
        return sum(a.elapsed_time(b) for a, b in self.events) / 1e3


class CallProfiler:
    """CUDA events around EVERY library call (side workloads, outside the
    timed regions): per-entry-point device time, launches and algorithmic
    work, for the kernel tables and rooflines of the side configs."""

    def __init__(self):
        self.events = {}
        self.work = {}

    def hook(self, name, args, run):
        import torch
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        rc = run()
        b.record()
        self.events.setdefault(name, []).append((a, b))
        self.work[name] = self.work.get(name, 0) + work_of(name, args)
        return rc

    def seconds(self, name: str) -> float:
        return sum(a.elapsed_time(b) for a, b in self.events.get(name, ())) / 1e3

    def table(self, wall_s: float, top: int = 5) -> dict:
        import torch
        torch.cuda.synchronize()
        rows = sorted(((self.seconds(n), n) for n in self.events), reverse=True)
        busy = sum(t for t, _ in rows)
        return {"wall_ms": wall_s * 1e3, "device_busy_ms": busy * 1e3,
                "launches": sum(len(v) for v in self.events.values()),
                "top": [{"entry_point": n, "ms": t * 1e3, "share_of_wall": t / wall_s if wall_s else None,
                         "launches": len(self.events[n]), **self.roofline(n, t)} for t, n in rows[:top]]}

    def roofline(self, name: str, secs: float) -> dict:
        bound = KERNEL_BOUND.get(name)
        if bound is None or not secs or not self.work.get(name):
            return {}
        kind, unit, scale = bound
        return {"bound": kind, "achieved": self.work[name] / secs / scale, "unit": unit}


def table_roofline(tab: dict, peaks: dict) -> dict:
    """Roofline of the largest-time kernel with a known bound in a kernel
    table (CallProfiler.table): achieved rate against the peak of its bound,
    and its share of the leg's wall time."""
    for t in tab.get("top", []):
        if "bound" in t and t["bound"] in peaks and t.get("achieved"):
            peak, src = peaks[t["bound"]]
            return {"bound": t["bound"], "kernel": t["entry_point"], "achieved": t["achieved"], "peak": peak,
                    "unit": t["unit"], "frac": t["achieved"] / peak, "share_of_wall": t["share_of_wall"],
                    "launches": t["launches"], "peak_source": src}
    return {"bound": None, "why": "no bounded kernel among the top entries"}


def work_of(name, args) -> int:
    """Algorithmic work of one call: bytes moved for the HBM-bound tensor-core
    line evaluations (r3_gr_matmul2_tc reads nops rows of 512 B and writes one
    per output row), u64 multiply-accumulates for the CUDA-core
    GR contractions."""
    if name in ("r3_gr_matmul2_tc", "r3_gr_matmul2_tc16"):
        w = 512 if name == "r3_gr_matmul2_tc" else 128
        p1, nv0, nv1, rows = args[3], int(args[2]), int(args[5]), int(args[9])
        return w * (rows + min(nv0, rows) + (min(nv1, rows) if p1 else 0))
    if name in ("r3_gr_matmul2_tc_multi", "r3_gr_matmul2_tc16_multi"):
        w = 512 if name == "r3_gr_matmul2_tc_multi" else 128
        nj, nv0, nv1, rows = int(args[0]), args[3], args[6], args[10]
        return sum(w * (int(rows[j]) + min(int(nv0[j]), int(rows[j])) + min(int(nv1[j]), int(rows[j])))
                   for j in range(nj))
    if name == "r3_gr_matmul_q_tc":
        # TMEM bytes the epilogue drains: eight 32-bit limb diagonals per
        # output u64, 64 words per row, one output per public matrix
        return 32 * 64 * int(args[2]) * int(args[5])
    if name == "r3_gr_matmul_k16_tc":
        return 32 * 64 * int(args[1])
    if name == "r3_prf_ctr":
        return -(-int(args[2]) // 2)                       # AES blocks
    if name == "r3_prf_bits_packed":
        return -(-int(args[2]) * int(args[3]) // 2)        # nbits x lanes words
    if name == "r3_ripple_msb":
        lanes, ell = int(args[6]), int(args[7])
        return 3 * (ell - 2) * lanes // 2                  # 3 words per gate and lane
    if name == "r3_ew_flat":
        n, b = int(args[1]), args[4]
        return 8 * n * (3 if b else 2)                     # bytes
    if name == "r3_u64_gemm_tc":
        npairs, K, M, N = int(args[0]), args[3], int(args[4]), int(args[5])
        return 2 * 36 * M * N * sum(int(K[p]) for p in range(npairs))
    if name in ("r3_vfy_base_fold_q8", "r3_vfy_base_fold_q16"):
        # useful accumulator updates as int8 limb ops: per block of B, every
        # party's B^2 s products and B z values per z array times one table
        # row of 64 coefficients (36 limb products x 2)
        import ctypes as C
        B = 8 if name.endswith("q8") else 16
        np_, N = int(args[0]), int(args[8])
        nz = (C.c_int * np_).from_address(int(args[5]))
        feats = np_ * B * B + B * sum(int(v) for v in nz)
        return 72 * 64 * feats * ((N + B - 1) // B)
    if name == "r3_vfy_level_fold":
        # per pair: h(1) and h(2), one outer product each for P0, two for P1/P2
        role, N, d = args[0], args[5], args[6]
        pairs = (int(N) + 1) // 2
        return pairs * (2 if role == 0 else 4) * int(d) * int(d)
    if name == "r3_gr_dotsum":
        rows, d = args[2], args[3]
        return int(rows) * int(d) * int(d)
    if name == "r3_gr_matmul":
        rows, d = args[5], args[6]
        return int(rows) * int(d) * int(d)
    return 0


TMEM_READ_B_PER_CLK = 64

KERNEL_BOUND = {
    "r3_gr_matmul2_tc": ("hbm", "GB/s", 1e9),
    "r3_gr_matmul2_tc16": ("hbm", "GB/s", 1e9),
    "r3_gr_matmul2_tc_multi": ("hbm", "GB/s", 1e9),
    "r3_gr_matmul2_tc16_multi": ("hbm", "GB/s", 1e9),
    "r3_ew_flat": ("hbm", "GB/s", 1e9),
    # the table kernels write four bytes per byte read and are paced by the
    # TMEM drain of their limb diagonals (ncu r05f)
    "r3_gr_matmul_q_tc": ("tmem", "TB/s TMEM read", 1e12),
    "r3_gr_matmul_k16_tc": ("tmem", "TB/s TMEM read", 1e12),
    "r3_u64_gemm_tc": ("tensor", "int8 TOP/s", 1e12),
    "r3_vfy_base_fold_q8": ("tensor", "int8 TOP/s", 1e12),
    "r3_vfy_base_fold_q16": ("tensor", "int8 TOP/s", 1e12),
    "r3_prf_ctr": ("aes", "G AES blocks/s", 1e9),
    "r3_prf_bits_packed": ("aes", "G AES blocks/s", 1e9),
    "r3_ripple_msb": ("aes", "G AES blocks/s", 1e9),
    "r3_vfy_level_fold": ("int-alu", "Tu64MAC/s", 1e12),
    "r3_gr_matmul": ("int-alu", "Tu64MAC/s", 1e12),
    "r3_gr_dotsum": ("int-alu", "Tu64MAC/s", 1e12),
}


def ncu_traffic(kernel: str) -> dict:
    """DRAM bytes of one ncu --set full capture of the kernel against that
    launch's algorithmic bytes (profiles/r01_traffic.json): traffic well
    above the algorithmic bytes would mean re-reads."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_traffic.json")) as f:
            j = json.load(f)
        k = j["r3::gr_matmul2_tc_kernel" if kernel == "r3_gr_matmul2_tc" else kernel]
        return {"traffic": k["dram_read_bytes"] + k["dram_write_bytes"],
                "traffic_algorithmic": k.get("algorithmic_bytes"),
                "traffic_launch": k.get("launch"), "traffic_source": j.get("source")}
    except (OSError, KeyError, ValueError):
        return {"traffic": None}


def hbm_peak() -> tuple[float, str]:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]) * 1e9, "MEASURED_PEAKS.json hbm_gbs (burst copy)"
    except (OSError, KeyError, ValueError):
        return 6.65e12, "fallback 6.65 TB/s (B200_PROFILING.md; MEASURED_PEAKS.json absent)"


INT8_DENSE_NOMINAL = 4.5e15


def int8_peak_ops(torch) -> float:
    """Measured dense int8 tensor throughput (cuBLASLt torch._int_mm, 8192^3)."""
    n = 8192
    a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
    torch._int_mm(a, b)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        torch._int_mm(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, 2 * n ** 3 / (e0.elapsed_time(e1) / 1e3))
    return best


def imad_peak_macs(torch, lib) -> float:
    """Measured u64-MAC ceiling of the integer pipe (r3_imad_peak)."""
    sink = torch.zeros(1, dtype=torch.int64, device="cuda")
    it = 4096
    lib.call("r3_imad_peak", 256, sink.data_ptr(), lib.stream())
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(3):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        lib.call("r3_imad_peak", it, sink.data_ptr(), lib.stream())
        b.record()
        torch.cuda.synchronize()
        secs = a.elapsed_time(b) / 1e3
        best = max(best, 148 * 8 * 256 * 8 * it / secs)
    return best


def run_b200(args):
    import torch
    import numpy as np

    from paper_2411_09287_b200 import _lib, verify
    from paper_2411_09287_b200.runtime import Session

    from paper_2411_09287_b200 import dist as pdist
    rank, world, local = pdist.init(args.dist_backend)
    _lib.load()

    N = 1 << args.log2n
    d = args.d
    R = verify.pick_r(N, 64, d, "lan") if args.R == "auto" else int(args.R)
    mulv, e2e = make_programs(N, d, R)

    def barrier():
        pdist.barrier()
        torch.cuda.synchronize()

    def step(i):
        sess = Session(seed=pdist.session_seed(rank, i), engine=args.engine)
        res = sess.run(mulv)
        return res

    for i in range(args.warmup):
        res = step(i)
        assert all(res), "honest verification rejected"

    timer = KernelTimer(args.profile_kernel)
    launches0 = _lib.load().r3_launch_count()
    _lib.CALL_HOOK = timer.hook
    _lib.CALL_HOOK_ONLY = timer.names
    barrier()
    with Clocks(local) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        wall0 = time.perf_counter()
        for i in range(args.steps):
            res = step(args.warmup + i)
        t1.record()
        barrier()
        wall = time.perf_counter() - wall0
    _lib.CALL_HOOK = None
    _lib.CALL_HOOK_ONLY = None
    launches = _lib.load().r3_launch_count() - launches0
    assert all(res)
    secs = pdist.max_over_ranks(t0.elapsed_time(t1) / 1e3)
    ms_per_step = secs / args.steps * 1e3
    value = N * world * args.steps / secs

    # roofline of the dominant kernel, timed live in the region above
    kt = timer.seconds()
    bound, r_unit, scale = KERNEL_BOUND.get(args.profile_kernel, ("int-alu", "Tu64MAC/s", 1e12))
    if bound == "hbm":
        peak, peak_src = hbm_peak()
        work_desc = "algorithmic bytes = 512 B x (rows written + rows read per operand) per launch"
    else:
        peak = imad_peak_macs(torch, _lib)
        peak_src = "measured in-run by r3_imad_peak (MEASURED_PEAKS.json has no integer peak)"
        work_desc = "algorithmic work = rows*d^2 u64 MACs per launch"
    achieved = timer.work / kt if kt else 0.0

    # end-to-end: host inputs in pinned memory (this rank's shard of the
    # global batch), opened product shards gathered to rank 0 over NCCL and
    # copied back to the host there
    def shard_inputs(r):
        g = np.random.default_rng(1000 + r)
        return (g.integers(0, 2**63, N, dtype=np.int64), g.integers(0, 2**63, N, dtype=np.int64))
    xv, yv = shard_inputs(rank)
    xh = torch.from_numpy(xv).pin_memory()
    yh = torch.from_numpy(yv).pin_memory()

    # the opened product of step i is copied D2H on a side stream into one of
    # two pinned buffers while step i + 1 runs; every copy completes inside
    # the timed region (the loop ends with a wait on the last one)
    out_host = [torch.empty(N * world, dtype=torch.int64, pin_memory=True) for _ in range(2)] \
        if rank == 0 else None
    d2h_stream = torch.cuda.Stream() if rank == 0 else None
    d2h_done = [None, None]

    from paper_2411_09287_b200._lib import StagedInput
    staged = {}

    def e2e_step(seed, slot, prefetch=False):
        # this step's input copies may have been started by the previous
        # step's verification (prefetch); every copy of a timed step is
        # inside the timed region
        pre = dict(staged)
        staged.clear()
        nxt = (lambda role, host: staged.__setitem__(role, StagedInput(host))) if prefetch else None
        z = Session(seed=seed).run(e2e, xh, yh, pre, nxt)[0]
        full = pdist.gather_outputs(z)
        if rank != 0:
            return None
        if d2h_done[slot] is not None:
            d2h_done[slot].synchronize()          # buffer free again
        if not full.is_cuda:                      # gloo gather (CPU test path)
            out_host[slot].copy_(full)
            d2h_done[slot] = None
            return out_host[slot]
        ready = torch.cuda.Event()
        ready.record()
        with torch.cuda.stream(d2h_stream):
            d2h_stream.wait_event(ready)
            out_host[slot].copy_(full, non_blocking=True)   # D2H into pinned memory
            full.record_stream(d2h_stream)
            ev = torch.cuda.Event()
            ev.record()
        d2h_done[slot] = ev
        return out_host[slot]

    def e2e_drain():
        if rank == 0:
            for ev in d2h_done:
                if ev is not None:
                    ev.synchronize()

    # two untimed steps (the second consumes the first's prefetched inputs),
    # so the timed loop starts with the allocator and copy streams warm
    e2e_step(pdist.session_seed(rank, 0, stream=1), 0, prefetch=True)
    e2e_step(pdist.session_seed(rank, 1 << 30, stream=1), 1)
    e2e_drain()
    barrier()
    e0 = time.perf_counter()
    for i in range(args.e2e_steps):
        out = e2e_step(pdist.session_seed(rank, 1 + i, stream=1), i % 2, prefetch=i + 1 < args.e2e_steps)
    e2e_drain()
    barrier()
    e2e_s = pdist.max_over_ranks(time.perf_counter() - e0)
    if rank == 0:
        got = out.numpy().view(np.uint64).reshape(world, N)
        for r in range(world):
            xs, ys = shard_inputs(r)
            assert np.array_equal(got[r], xs.view(np.uint64) * ys.view(np.uint64)), "e2e product mismatch"

    # the headline step's whole-step kernel table and the per-party rate
    # (rank 0; outside the timed region): one session under the per-call
    # profiler, and one session with joint kernels off -- every party's
    # local kernels launched per party, pairwise PRF draws and m-derived
    # line evaluations still shared
    step_kernels = per_party = None
    if rank == 0 and not args.no_step_profile:
        cp = CallProfiler()
        _lib.CALL_HOOK = cp.hook
        torch.cuda.synchronize()
        tp = time.perf_counter()
        Session(seed=pdist.session_seed(rank, 1 << 20)).run(mulv)
        torch.cuda.synchronize()
        _lib.CALL_HOOK = None
        step_kernels = cp.table(time.perf_counter() - tp)
        # one warm-up session (first-use allocations of the per-party
        # launches), then the median of three
        Session(seed=pdist.session_seed(rank, (1 << 20) + 1), joint=False).run(mulv)
        pps = []
        for j in range(3):
            a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a_ev.record()
            ok = Session(seed=pdist.session_seed(rank, (1 << 20) + 2 + j), joint=False).run(mulv)
            b_ev.record()
            torch.cuda.synchronize()
            assert all(ok)
            pps.append(a_ev.elapsed_time(b_ev) / 1e3)
        pp = statistics.median(pps)
        per_party = {"value": N / pp, "unit": UNIT, "ms_per_step": pp * 1e3,
                     "what": "one session with joint kernels off (Session(joint=False)): each simulated "
                             "party launches its own kernels; the headline's joint launches batch the "
                             "three parties' local work, which a one-party-per-host deployment cannot"}

    # side configs, every rank; sharded over the
    # ranks, outputs all-gathered to rank 0 and checked there
    side = {}
    if args.matmul_n:
        side["matmul"] = matmul_c3(args.matmul_n, 3, rank, world, args.matmul_verified_rows)
    if args.relu_log2n:
        side["relu"] = relu_rates(1 << args.relu_log2n, 16, 5, rank, world)
    if args.relu_sweep_log2n:
        # weak scaling: 2^L lanes per GPU
        side["relu_sweep"] = relu_rates((1 << args.relu_sweep_log2n) * world, 16, 3, rank, world)
    if args.mlp_batch:
        side["mlp"] = ppml_rates("mlp", args.mlp_batch, args.mlp_verified_batch, rank, world)
    if args.lenet_batch:
        side["lenet"] = ppml_rates("lenet", args.lenet_batch, args.lenet_verified_batch, rank, world,
                                   args.lenet_batch)
    if world == 1 and args.mulv_sweep:
        variants = [tuple(None if x == "auto" else int(x) for x in v.split(":"))
                    for v in args.mulv_variants.split(",") if v]
        side["mulv_sweep"] = mulv_sweep([int(v) for v in args.mulv_sweep.split(",")], d, variants=variants)

    if rank != 0:
        pdist.finalize()
        return
    if "relu" in side or "relu_sweep" in side:
        prf_peak = prf_peak_blocks(torch, _lib)
        for key in ("relu", "relu_sweep"):
            r = side.get(key)
            if r and "aes_blocks_per_lane" in r:
                ach = r["exec"] * r["aes_blocks_per_lane"]
                r["roofline"] = {"bound": "aes", "leg": "exec", "achieved": ach / 1e9, "peak": prf_peak / 1e9,
                                 "unit": "G AES blocks/s", "frac": ach / prf_peak,
                                 "peak_source": "measured in-run: r3_prf_ctr bulk keystream rate (2^26 blocks)",
                                 "work": "AES blocks of keystream the protocol consumes per lane (every "
                                         "distinct pairwise stream up to its final offset) x lanes / exec time"}
    # C4 / C5: roofline of each leg's dominant bounded kernel (its kernel
    # table, CUDA events around every call of one extra session)
    peaks = None
    for key in ("mlp", "lenet"):
        r = side.get(key)
        if not r:
            continue
        if peaks is None:
            peaks = {"hbm": (hbm_peak()[0] / 1e9, "MEASURED_PEAKS.json hbm_gbs (burst copy)"),
                     "aes": (prf_peak_blocks(torch, _lib) / 1e9, "measured in-run: r3_prf_ctr bulk rate"),
                     "tensor": (INT8_DENSE_NOMINAL / 1e12, "nominal dense int8 (4.5 POPS)"),
                     "int-alu": (imad_peak_macs(torch, _lib) / 1e12, "measured in-run: r3_imad_peak")}
        rl = {}
        for leg in ("exec", "verified"):
            tab = r.get(leg + "_kernels")
            if tab:
                rl[leg] = table_roofline(tab, peaks)
        if rl:
            r["roofline"] = rl
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic: PRF-generated (AES-128-CTR) random shares, distinct seed per rank and step",
        "config": {"workload": "mulv: batched 3PC Pi_mul + GR(2^64,d) batch verification "
                               "(tests/test_acceptance.py:124-136), 3 parties per GPU",
                   "N_per_gpu": N, "sweep_point": "2^28 over 8 GPUs = 2^25 per GPU (config 2's sweep "
                                                  "end, weak scaling); 2^20..2^26 on one GPU in mulv_sweep",
                   "ell": 64, "d": d, "R": R, "engine": args.engine,
                   "l2": f"inputs larger than L2 ({N * 8 * 12 / 2**20:.0f} MiB of shares per step)",
                   "parallelism": f"weak dp{world}: element batch sharded, one 3-party session per rank "
                                  f"shard, NCCL gather of opened outputs"},
        "roofline": {"bound": bound, "kernel": args.profile_kernel,
                     "achieved": achieved / scale, "peak": peak / scale, "unit": r_unit,
                     "frac": achieved / peak if peak else None, **ncu_traffic(args.profile_kernel),
                     "launches": timer.launches, "kernel_s_per_step": kt / args.steps,
                     "kernel_share_of_step": kt / secs if secs else None,
                     "peak_source": peak_src + "; " + work_desc},
        "e2e": {"value": N * world * args.e2e_steps / e2e_s, "unit": UNIT,
                "h2d_bytes_per_step": 2 * N * 8 * world, "d2h_bytes_per_step": N * 8 * world,
                "steps": args.e2e_steps, "warmup": 2,
                "path": "per rank: pinned host shard -> Session.run (PRE, ONLINE, Pi_mulv, open) -> "
                        "NCCL all-gather of the opened shards -> rank 0 host (the H2D of step i + 1 starts "
                        "when step i's verification starts and the D2H of step i overlaps step i + 1, both "
                        "on a copy stream; every copy of the timed steps is inside the timed region)"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "wall_s_timed": wall,
    }
    if step_kernels is not None:
        line["step_kernels"] = step_kernels
        line["per_party_rate"] = per_party
        # the step's largest-time bounded kernel (the base fold is tensor /
        # converter bound, so its fraction is of nominal dense int8)
        top = step_kernels["top"][0]["entry_point"] if step_kernels.get("top") else None
        tpeaks = {"hbm": (hbm_peak()[0] / 1e9, "MEASURED_PEAKS.json hbm_gbs (burst copy)"),
                  "tensor": (INT8_DENSE_NOMINAL / 1e12, "nominal dense int8 (4.5 POPS)")}
        sm_mhz = line["clocks"].get("sm_mhz") or line["clocks"].get("sm_max_mhz")
        if sm_mhz:
            nsm = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
            tpeaks["tmem"] = (TMEM_READ_B_PER_CLK * nsm * sm_mhz * 1e6 / 1e12,
                              f"TMEM read {TMEM_READ_B_PER_CLK} B/clk/SM (B300_MICROARCH.md LDTM throughput, "
                              f"measured on B300) x {nsm} SMs x {sm_mhz:.0f} MHz (median SM clock of the timed region)")
        line["roofline_step_top"] = dict(table_roofline(step_kernels, tpeaks), top_entry_point=top)
    line.update(side)
    if world == 1 and not args.no_cpu_baseline:
        # same-run CPU baselines (rank 0, N = 1): the unmodified reference on
        # every host core, one leg per config
        line["cpu_baseline"] = cpu_leg("mulv", args.cpu_seconds / 2)
        legs = {"relu": ("relu_exec", "relu_verified"), "matmul": ("matmul",),
                "mlp": ("mlp_exec", "mlp_verified"), "lenet": ("lenet_exec",)}
        for key, works in legs.items():
            if key in line:
                cb = {w: cpu_leg(w, args.cpu_seconds / 2) for w in works}
                line[key]["cpu_baseline"] = cb if len(cb) > 1 else cb[works[0]]
    print(json.dumps(line), flush=True)
    pdist.finalize()


def run_reference(args):
    """--impl reference: the reference's own CPU implementation of the path
    (the unmodified ring3pc from baseline/_ref, bench_cpu.py) on the host
    cores, rank 0 only; each step one bounded parallel round of mulv
    sessions.  Falls back to the oracle port if the reference is absent."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    import bench_cpu
    ex = bench_cpu.pool()
    for _ in range(args.warmup):
        bench_cpu.measure("mulv", budget_s=0.0, max_rounds=1, executor=ex)
    vals = [bench_cpu.measure("mulv", budget_s=0.0, max_rounds=1, executor=ex) for _ in range(args.steps)]
    ex.shutdown()
    v = statistics.median(x["value"] for x in vals)
    cb = dict(vals[-1])
    cb["value"] = v
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u64", "impl": "reference",
            "data": "synthetic: PRF-generated random shares",
            "config": {"workload": "mulv: batched 3PC Pi_mul + GR(2^64,d) batch verification "
                                   "(tests/test_acceptance.py:124-136), the reference's own CPU code",
                       "N_per_session": bench_cpu.WORKLOADS["mulv"][0], "d": args.d, "ell": 64,
                       "R": "pick_r(lan)"},
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
