"""Micro-benchmark of the GR contraction kernels (CUDA events, warm)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2411_09287_b200 import grvec, _lib
from paper_2411_09287_b200.rings import modulus_for_degree

def timeit(fn, reps=10):
    fn(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps / 1e3

mod = modulus_for_degree(64)
for rows in (1 << 16, 1 << 20, 1 << 22):
    A0 = torch.randint(-2**62, 2**62, (rows, 64), dtype=torch.int64, device="cuda")
    A1 = torch.randint(-2**62, 2**62, (rows, 64), dtype=torch.int64, device="cuda")
    c = torch.randint(-2**62, 2**62, (1, 64), dtype=torch.int64, device="cuda")
    M = grvec.gr_mulmat(c, mod)
    out = grvec.empty((rows, 64))
    tc = lambda: _lib.call("r3_gr_matmul2_tc", A0.data_ptr(), 64, rows, A1.data_ptr(), 64, rows, M.data_ptr(), M.data_ptr(), out.data_ptr(), rows, (1 << 64) - 1, _lib.stream())
    cc = lambda: grvec.gr_matmul(grvec.lin((1, A1), (-1, A0)), M, rows, 64, 64, C_add=grvec.lin((1, A0)), out=out)
    ttc, tcc = timeit(tc), timeit(cc)
    macs = rows * 64 * 64
    byts = rows * 64 * 8 * 3
    print(f"rows={rows:8d}  tc {ttc*1e3:8.3f} ms ({macs/ttc/1e12:6.2f} Tu64MAC/s, {byts/ttc/1e9:7.1f} GB/s)   cuda-core {tcc*1e3:8.3f} ms ({macs/tcc/1e12:6.2f} Tu64MAC/s)")
    F = A0; G = A1
    acc = grvec.dotsum_acc(64)
    ds = lambda: grvec.dotsum_add(acc, grvec.lin((1, F)), grvec.lin((1, G)), rows, 64)
    tds = timeit(ds)
    print(f"             dotsum cuda-core {tds*1e3:8.3f} ms ({macs/tds/1e12:6.2f} Tu64MAC/s)")
    # pipelined tensor-core: f0.Ma + f1.Mb over even/odd rows of a 2*rows array
    X = torch.randint(-2**62, 2**62, (2 * rows, 64), dtype=torch.int64, device="cuda")
    ev, od = X[0::2], X[1::2]
    o2 = grvec.empty((rows, 64))
    t2 = lambda: _lib.call("r3_gr_matmul2_tc", ev.data_ptr(), 128, rows, od.data_ptr(), 128, rows, M.data_ptr(), M.data_ptr(), o2.data_ptr(), rows, (1 << 64) - 1, _lib.stream())
    tt2 = timeit(t2)
    print(f"             matmul2_tc (2 operands) {tt2*1e3:8.3f} ms ({2*macs/tt2/1e12:6.2f} Tu64MAC/s, {rows*64*8*3/tt2/1e9:7.1f} GB/s)")
    t1 = lambda: _lib.call("r3_gr_matmul2_tc", A0.data_ptr(), 64, rows, None, 0, 0, M.data_ptr(), None, o2.data_ptr(), rows, (1 << 64) - 1, _lib.stream())
    tt1 = timeit(t1)
    print(f"             matmul2_tc (1 operand)  {tt1*1e3:8.3f} ms ({macs/tt1/1e12:6.2f} Tu64MAC/s, {rows*64*8*2/tt1/1e9:7.1f} GB/s)")
