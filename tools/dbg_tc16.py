"""d = 16 tensor-core line evaluation against the oracle at multi-wave sizes (debug aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import gr as ogr
from paper_2411_09287_b200 import grvec, host, _lib
from paper_2411_09287_b200.rings import modulus_for_degree
d = 16
mod = modulus_for_degree(d)
for rows in (148 * 128 + 1, 300001, 1000000):
    rng = np.random.default_rng(rows)
    X = rng.integers(0, 2**64, (rows, d), dtype=np.uint64)
    z = rng.integers(0, 2**64, (1, d), dtype=np.uint64)
    Xd = grvec.dev(X)
    Mb = grvec.gr_mulmat(grvec.dev(z), mod)
    out1 = grvec.empty((rows, d))
    _lib.call("r3_gr_matmul2_tc16", Xd.data_ptr(), d, rows, None, 0, 0, Mb.data_ptr(), None, out1.data_ptr(), rows, (1 << 64) - 1, _lib.stream())
    want = ogr.mul(X, z, 64, d)
    got = host(out1)
    bad = np.argwhere(got != want)
    print(rows, "bad", len(bad), "rows", np.unique(bad[:, 0])[:8], "tiles", np.unique(bad[:, 0] // 128)[:10], "cols", np.unique(bad[:, 1]))
