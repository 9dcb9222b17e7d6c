"""Host vs device time of the secure-ReLU program, plus per-entry GPU time."""
import collections, gc, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, bench
from paper_2411_09287_b200.runtime import Session
from paper_2411_09287_b200 import _lib
N = 1 << int(sys.argv[1]); d = 16
engine = sys.argv[2] if len(sys.argv) > 2 else "coop"
rng = np.random.default_rng(1)
xv = np.trunc(rng.normal(0, 4, N) * 2 ** 16).astype(np.int64)
xh = torch.from_numpy(xv).pin_memory()
prog = bench.make_relu_program(N, d)
for check in (False, True):
    for nogc in (False, True):
        if nogc:
            gc.disable()
        for i in range(5):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            t = time.perf_counter(); e0.record()
            Session(seed=10 + i, engine=engine).run(prog, xh, check)
            e1.record(); th = time.perf_counter() - t
            torch.cuda.synchronize(); tw = time.perf_counter() - t
            print("check" if check else "exec", "nogc" if nogc else "gc", i, f"host {th*1e3:.1f} wall {tw*1e3:.1f} dev {e0.elapsed_time(e1):.1f} ms", flush=True)
        gc.enable()
    ev = []
    def hook(name, args, run):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); rc = run(); e.record(); ev.append((name, s, e)); return rc
    _lib.CALL_HOOK = hook
    Session(seed=99, engine=engine).run(prog, xh, check)
    _lib.CALL_HOOK = None
    torch.cuda.synchronize()
    tot = collections.Counter(); cnt = collections.Counter()
    for name, s, e in ev:
        tot[name] += s.elapsed_time(e); cnt[name] += 1
    for k, v in tot.most_common(12):
        print(f"   {k:28s} {v:8.2f} ms  x{cnt[k]}")
