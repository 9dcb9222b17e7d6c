"""Per-entry-point GPU time breakdown of one mulv step (CUDA events around
every library call, on the launching stream).  Diagnostic only.

    python tools/breakdown.py --log2n 22 --d 64
"""

import argparse
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_09287_b200 import _lib, verify  # noqa: E402
from paper_2411_09287_b200.runtime import Session  # noqa: E402


def _matmul_program(n):
    import numpy as np
    from paper_2411_09287_b200 import gates
    from paper_2411_09287_b200.sharing import Ring, shc_input_mask, shc_input_online
    from paper_2411_09287_b200.transport import Phase
    rng = np.random.default_rng(3)
    enc = lambda a: torch.from_numpy(np.trunc(a * 2 ** 16).astype(np.int64)).pin_memory()
    Xh, Wh = enc(rng.normal(0, 1, (n, n))), enc(rng.normal(0, 1 / 64, (n, n)))

    def prog(party):
        ring = Ring(64)
        party.enter_phase(Phase.PRE)
        xm = shc_input_mask(party, 2, n * n, ring)
        wm = shc_input_mask(party, 1, n * n, ring)
        tr = gates.trunc_prepare(party, n * n, 16, ring)
        g = gates.matmul_prepare(party, xm, wm, n, n, n, out_mask=tr.rx_mask)
        party.round_barrier()
        party.enter_phase(Phase.ONLINE)
        X = shc_input_online(party, 2, Xh.reshape(-1) if party.role == 2 else None, xm, n * n, ring, "X")
        W = shc_input_online(party, 1, Wh.reshape(-1) if party.role == 1 else None, wm, n * n, ring, "W")
        gates.trunc_online(party, gates.matmul_finish(party, g, X, W, log=False), tr)
        party.round_barrier()
        party.enter_phase(Phase.POST)
        party.freeze_logs()
    return prog


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2n", type=int, default=22)
    ap.add_argument("--d", type=int, default=64)
    ap.add_argument("--engine", default="coop")
    ap.add_argument("--top-calls", default="", help="kernel name: print its 15 slowest calls with a stack hint")
    ap.add_argument("--prog", default="mulv", choices=["mulv", "relu", "relu-exec", "matmul"])
    a = ap.parse_args()
    N = 1 << a.log2n
    R = verify.pick_r(N, 64, a.d)
    if a.prog == "mulv":
        mulv, _ = bench.make_programs(N, a.d, R)
        args = ()
    elif a.prog == "matmul":              # config C3 at n = 2^(log2n / 2)
        mulv = _matmul_program(1 << (a.log2n // 2))
        args = ()
    else:
        import numpy as np
        mulv = bench.make_relu_program(N, a.d)
        xv = np.trunc(np.random.default_rng(1).normal(0, 4, N) * 2 ** 16).astype(np.int64)
        args = (torch.from_numpy(xv).pin_memory(), a.prog == "relu")
    for i in range(2):
        Session(seed=i, engine=a.engine).run(mulv, *args)
    torch.cuda.synchronize()
    ev = []

    def hook(name, args, run):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        rc = run()
        e.record()
        where = ""
        if name == a.top_calls:
            import traceback
            fr = [f for f in traceback.extract_stack()[:-2] if "paper_2411_09287_b200" in f.filename]
            where = " <- ".join(f"{os.path.basename(f.filename)}:{f.lineno}:{f.name}" for f in fr[-3:][::-1])
        ev.append((name, s, e, where, [x for x in args if isinstance(x, int)][:4]))
        return rc

    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    t0.record()
    _lib.CALL_HOOK = hook
    Session(seed=99, engine=a.engine).run(mulv, *args)
    _lib.CALL_HOOK = None
    t1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    step = t0.elapsed_time(t1)
    tot = collections.Counter()
    cnt = collections.Counter()
    for name, s, e, _w, _a in ev:
        tot[name] += s.elapsed_time(e)
        cnt[name] += 1
    busy = sum(tot.values())
    print(f"{a.prog} N=2^{a.log2n} d={a.d} R={R}: step {step:.1f} ms (wall {wall*1e3:.1f} ms), "
          f"library GPU time {busy:.1f} ms in {len(ev)} calls")
    for k, v in tot.most_common():
        print(f"  {k:24s} {v:9.2f} ms {100 * v / step:5.1f}%  calls={cnt[k]}")
    if a.top_calls:
        sites = collections.Counter()
        for name, s, e, w, ia in ev:
            if name == a.top_calls:
                sites[w] += s.elapsed_time(e)
        print(f"{a.top_calls} by call site:")
        for w, v in sites.most_common(15):
            print(f"  {v:8.3f} ms  {w}")
        calls = sorted(((s.elapsed_time(e), w, ia) for name, s, e, w, ia in ev if name == a.top_calls),
                       key=lambda t: -t[0])
        print(f"{a.top_calls} slowest calls (int args):")
        for t, w, ia in calls[:12]:
            print(f"  {t:8.3f} ms  {ia}  {w.split(' <- ')[-1] if w else ''}")


if __name__ == "__main__":
    main()
