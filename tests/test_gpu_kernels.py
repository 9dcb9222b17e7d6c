"""Kernel-level parity: tensor-core and CUDA-core GR contractions against the
numpy oracle (oracle/gr.py) and against each other."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rand(rng, shape):
    return rng.integers(0, 2**64, shape, dtype=np.uint64)


@pytest.mark.parametrize("rows", [1, 127, 128, 129, 1000, 40000])
def test_gr_matmul_cuda_core_matches_oracle(cuda, rows):
    from oracle import gr as ogr
    from paper_2411_09287_b200 import grvec, host
    from paper_2411_09287_b200.rings import modulus_for_degree
    mod = modulus_for_degree(64)
    rng = np.random.default_rng(rows)
    a0 = _rand(rng, (rows, 64))
    a1 = _rand(rng, (rows, 64))
    c = _rand(rng, (1, 64))
    A0, A1, Cc = grvec.dev(a0), grvec.dev(a1), grvec.dev(c)
    M = grvec.gr_mulmat(Cc, mod)
    with np.errstate(over="ignore"):
        want = ogr.mul(a1 - a0, c, 64, 64) + a0
    ref = grvec.gr_matmul(grvec.lin((1, A1), (-1, A0)), M, rows, 64, 64, C_add=grvec.lin((1, A0)))
    np.testing.assert_array_equal(host(ref), want)


def test_gr_dotsum_matches_oracle(cuda):
    from oracle import gr as ogr
    from paper_2411_09287_b200 import grvec, host
    from paper_2411_09287_b200.rings import modulus_for_degree
    rng = np.random.default_rng(5)
    for d in (2, 8, 16, 64):
        mod = modulus_for_degree(d)
        f = _rand(rng, (3001, d))
        g = _rand(rng, (3001, d))
        got = host(grvec.gr_dot(grvec.dev(f), grvec.dev(g), 64, mod))
        np.testing.assert_array_equal(got, ogr.dot(f, g, 64, d))


def test_gr_mul_and_powers_match_oracle(cuda):
    from oracle import gr as ogr
    from paper_2411_09287_b200 import grvec, host
    from paper_2411_09287_b200.rings import modulus_for_degree
    rng = np.random.default_rng(9)
    for d in (1, 2, 4, 8, 16, 32, 64):
        mod = modulus_for_degree(d)
        a = _rand(rng, (77, d))
        b = _rand(rng, (77, d))
        np.testing.assert_array_equal(host(grvec.gr_mul(grvec.dev(a), grvec.dev(b), 64, mod)),
                                      ogr.mul(a, b, 64, d))
        r = _rand(rng, (1, d))
        np.testing.assert_array_equal(host(grvec.gr_powers(grvec.dev(r), 300, 64, mod)),
                                      ogr.powers(r, 300, 64, d))


@pytest.mark.parametrize("d,rows", [(64, 1), (64, 128), (64, 129), (64, 5000), (64, 70001),
                                    (16, 1), (16, 255), (16, 4097), (16, 300001)])
def test_gr_matmul2_tc_line_eval(cuda, d, rows):
    """Pipelined tensor-core contraction: f0 + (f1 - f0) z = f0.M(1-z) + f1.M(z),
    with even/odd row views and the odd-length zero pad (verify.py:220-240);
    d = 64 (r3_gr_matmul2_tc) and d = 16 (r3_gr_matmul2_tc16)."""
    from oracle import gr as ogr
    from paper_2411_09287_b200 import grvec, host, _lib
    from paper_2411_09287_b200.rings import modulus_for_degree
    mod = modulus_for_degree(d)
    fn = "r3_gr_matmul2_tc" if d == 64 else "r3_gr_matmul2_tc16"
    rng = np.random.default_rng(rows + 7 + d)
    X = _rand(rng, (rows, d))
    z = _rand(rng, (1, d))
    Xd = grvec.dev(X)
    one = np.zeros((1, d), dtype=np.uint64)
    one[0, 0] = 1
    with np.errstate(over="ignore"):
        Ma = grvec.gr_mulmat(grvec.dev(one - z), mod)
    Mb = grvec.gr_mulmat(grvec.dev(z), mod)
    n0, n1 = (rows + 1) // 2, rows // 2
    ev, od = Xd[0::2], Xd[1::2]
    out = grvec.empty((n0, d))
    _lib.call(fn, ev.data_ptr(), ev.stride(0), n0, od.data_ptr() if n1 else Xd.data_ptr(),
              od.stride(0) if n1 > 1 else 2 * d, n1, Ma.data_ptr(), Mb.data_ptr(), out.data_ptr(), n0,
              (1 << 64) - 1, _lib.stream())
    f0 = X[0::2]
    f1 = np.zeros_like(f0)
    f1[:n1] = X[1::2]
    with np.errstate(over="ignore"):
        want = ogr.mul(f1 - f0, z, 64, d) + f0
    np.testing.assert_array_equal(host(out), want)
    # single-operand form
    out1 = grvec.empty((rows, d))
    _lib.call(fn, Xd.data_ptr(), d, rows, None, 0, 0, Mb.data_ptr(), None, out1.data_ptr(),
              rows, (1 << 64) - 1, _lib.stream())
    np.testing.assert_array_equal(host(out1), ogr.mul(X, z, 64, d))
    # width-1 ring (the boolean log's GR(2, d)): masked output
    if d == 16:
        Xb = X & np.uint64(1)
        outb = grvec.empty((rows, d))
        _lib.call(fn, grvec.dev(Xb).data_ptr(), d, rows, None, 0, 0, Mb.data_ptr(), None, outb.data_ptr(),
                  rows, 1, _lib.stream())
        np.testing.assert_array_equal(host(outb), ogr.mul(Xb, z, 64, d) & np.uint64(1))


@pytest.mark.parametrize("d", [64, 16])
def test_gr_matmul2_tc_multi_matches_single_launches(cuda, d):
    """r3_gr_matmul2_tc_multi / _tc16_multi (several line evaluations
    sharing M(1 - z), M(z) in one launch: ragged job sizes, odd lengths, a
    one-row job, strided even/odd views) equals one single-job launch per
    job."""
    from paper_2411_09287_b200 import grvec, host
    from paper_2411_09287_b200.rings import modulus_for_degree
    mod = modulus_for_degree(d)
    rng = np.random.default_rng(77 + d)
    z = _rand(rng, (1, d))
    one = np.zeros((1, d), dtype=np.uint64)
    one[0, 0] = 1
    with np.errstate(over="ignore"):
        Ma = grvec.gr_mulmat(grvec.dev(one - z), mod)
    Mb = grvec.gr_mulmat(grvec.dev(z), mod)
    jobs = []
    for rows in (2, 3, 257, 4096, 70001, 129, 1000, 9, 33):
        Xd = grvec.dev(_rand(rng, (rows, d)))
        jobs.append((Xd[0::2], Xd[1::2], (rows + 1) // 2, rows // 2))
    got = grvec.rows_times2_batch(jobs, Ma, Mb, 64)
    for (ev, od, n0, n1), g in zip(jobs, got):
        want = grvec.rows_times(ev, Ma, n0, 64, P1=od, M1=Mb, nvalid=(n0, n1))
        np.testing.assert_array_equal(host(g), host(want))


@pytest.mark.parametrize("rows,q", [(1, 4), (129, 4), (5000, 3), (70001, 4), (1 << 18, 2), (300, 1)])
def test_gr_matmul_q_tc(cuda, rows, q):
    """r3_gr_matmul_q_tc: one operand times q public matrices in one pass
    (strided rows, partial last tile) against the oracle GR product."""
    from oracle import gr as ogr
    from paper_2411_09287_b200 import grvec, host
    from paper_2411_09287_b200.rings import modulus_for_degree
    d = 64
    mod = modulus_for_degree(d)
    rng = np.random.default_rng(rows + q)
    X = _rand(rng, (2 * rows, d))
    zs = [_rand(rng, (1, d)) for _ in range(q)]
    Xd = grvec.dev(X)[0::2]                       # strided rows, as the even half of a level
    outs = [grvec.empty((rows, d)) for _ in range(q)]
    grvec.rows_times_multi(Xd, [grvec.gr_mulmat(grvec.dev(z), mod) for z in zs], rows, 64, outs)
    for z, o in zip(zs, outs):
        np.testing.assert_array_equal(host(o), ogr.mul(X[0::2], z, 64, d))
    outs63 = [grvec.empty((rows, d)) for _ in range(q)]
    grvec.rows_times_multi(Xd, [grvec.gr_mulmat(grvec.dev(z), mod) for z in zs], rows, 63, outs63)
    np.testing.assert_array_equal(host(outs63[-1]), ogr.mul(X[0::2], zs[-1], 64, d) & np.uint64((1 << 63) - 1))


@pytest.mark.parametrize("rows", [1, 129, 5000, 1 << 17])
def test_gr_matmul_k16_tc(cuda, rows):
    """r3_gr_matmul_k16_tc (y-side level-4 rows, K = 16 byte-limb GEMM)
    against its definition sum_a y[16j + a] K[a] (numpy, wrapping u64) and
    against r3_vfy_line_b_const with blocks of sixteen."""
    from paper_2411_09287_b200 import _lib, grvec, host
    from paper_2411_09287_b200._lib import call, ptr, stream
    import ctypes as C
    rng = np.random.default_rng(rows)
    Y = _rand(rng, (rows * 16,))
    K = _rand(rng, (16, 64))
    yd, kd = grvec.dev(Y), grvec.dev(K)
    out = grvec.empty((rows, 64))
    call("r3_gr_matmul_k16_tc", ptr(yd), rows, ptr(kd), ptr(out), (1 << 64) - 1, stream())
    want = np.zeros((rows, 64), dtype=np.uint64)
    with np.errstate(over="ignore"):
        for a in range(16):
            want += Y[a::16][:, None] * K[a][None, :]
    np.testing.assert_array_equal(host(out), want)
    ref = grvec.empty((rows, 64))
    P = C.c_void_p * 1
    call("r3_vfy_line_b_const", 16, 1, P(ptr(yd)), rows * 16, 1, 0, 1, ptr(kd), 64, P(ptr(ref)),
         (1 << 64) - 1, stream())
    np.testing.assert_array_equal(host(ref), want)
    out63 = grvec.empty((rows, 64))
    call("r3_gr_matmul_k16_tc", ptr(yd), rows, ptr(kd), ptr(out63), (1 << 63) - 1, stream())
    np.testing.assert_array_equal(host(out63), want & np.uint64((1 << 63) - 1))
    assert _lib is not None


@pytest.mark.parametrize("L,n,nterms", [(1, 16, 1), (45, 64, 2), (1000, 32, 3), (4099, 64, 2)])
def test_lane16_fold_and_line_match_definitions(cuda, L, n, nterms):
    """r3_vfy_lane16_fold / _line (dot logs with n % 16 == 0, d = 16) against
    their definitions: acc[a*16+b] = sum_l pw[l] sum_j sum_t c_t x_t[16j+a][l]
    y_t[16j+b][l]; level-4 rows sum_a kappa_a x[16j+a][l] (times pw[l] in GR
    on the x side, the oracle's GR product)."""
    from oracle import gr as ogr
    from paper_2411_09287_b200 import grvec, host
    from paper_2411_09287_b200._lib import call, ptr, stream
    from paper_2411_09287_b200.rings import modulus_for_degree
    import ctypes as C
    d = 16
    mod = modulus_for_degree(d)
    rng = np.random.default_rng(L * 7 + n)
    xs = [_rand(rng, (n, L)) for _ in range(nterms)]
    ys = [_rand(rng, (n, L)) for _ in range(nterms)]
    coef = [1, -1, 2][:nterms]
    pw = _rand(rng, (L, d))
    xd, yd, pwd = [grvec.dev(x) for x in xs], [grvec.dev(y) for y in ys], grvec.dev(pw)
    acc = grvec.empty((256, d))
    P = lambda ts: (C.c_void_p * len(ts))(*[ptr(t) for t in ts])
    call("r3_vfy_lane16_fold", nterms, (C.c_int64 * nterms)(*coef), P(xd), P(yd), L, n, ptr(pwd), d,
         ptr(acc), stream())
    want = np.zeros((256, d), dtype=np.uint64)
    with np.errstate(over="ignore"):
        S = np.zeros((256, L), dtype=np.uint64)
        for t in range(nterms):
            cf = np.uint64(coef[t] & ((1 << 64) - 1))
            for j in range(0, n, 16):
                for a in range(16):
                    for b in range(16):
                        S[a * 16 + b] += cf * xs[t][j + a] * ys[t][j + b]
        for q in range(256):
            want[q] = (S[q][:, None] * pw).sum(axis=0, dtype=np.uint64)
    np.testing.assert_array_equal(host(acc), want)
    kappa = _rand(rng, (16, d))
    kd = grvec.dev(kappa)           # device operands stay referenced until the launches ran
    rows = L * (n // 16)
    outs = [grvec.empty((rows, d)) for _ in range(2)]
    for pow_side, o in ((0, outs[0]), (1, outs[1])):
        call("r3_vfy_lane16_line", pow_side, 1, P(xd[:1]), L, n, ptr(pwd) if pow_side else None,
             ptr(kd), mod.lowterms_mask, d, P([o]), (1 << 64) - 1, stream())
    u = np.zeros((L, n // 16, d), dtype=np.uint64)
    with np.errstate(over="ignore"):
        for j in range(n // 16):
            for a in range(16):
                u[:, j] += xs[0][16 * j + a][:, None] * kappa[a][None, :]
    np.testing.assert_array_equal(host(outs[0]).reshape(L, n // 16, d), u)
    prod = ogr.mul(u.reshape(-1, d), np.repeat(pw, n // 16, axis=0), 64, d)
    np.testing.assert_array_equal(host(outs[1]), prod)


@pytest.mark.parametrize("N", [1, 16, 1000, 70001])
def test_mul16_line_matches_definition(cuda, N):
    """r3_vfy_mul16_line (d = 16 multiplication-log level-4 rows, blocks of
    sixteen, ragged tail): row j = sum_a coef[a] x[16j + a], times pw16[j]
    with the oracle's GR product on the x side."""
    from oracle import gr as ogr
    from paper_2411_09287_b200 import grvec, host
    from paper_2411_09287_b200._lib import call, ptr, stream
    from paper_2411_09287_b200.rings import modulus_for_degree
    import ctypes as C
    d = 16
    mod = modulus_for_degree(d)
    rng = np.random.default_rng(N)
    rows = (N + 15) // 16
    X = _rand(rng, (N,))
    coef = _rand(rng, (16, d))
    pw = _rand(rng, (rows, d))
    xd, cd, pd = grvec.dev(X), grvec.dev(coef), grvec.dev(pw)
    P = lambda ts: (C.c_void_p * len(ts))(*[ptr(t) for t in ts])
    Xp = np.zeros(rows * 16, dtype=np.uint64)
    Xp[:N] = X
    u = np.zeros((rows, d), dtype=np.uint64)
    with np.errstate(over="ignore"):
        for a in range(16):
            u += Xp[a::16][:, None] * coef[a][None, :]
    for pow_side, want in ((0, u), (1, ogr.mul(u, pw, 64, d))):
        o = grvec.empty((rows, d))
        call("r3_vfy_mul16_line", pow_side, 1, P([xd]), N, ptr(pd) if pow_side else None, ptr(cd),
             mod.lowterms_mask, d, P([o]), (1 << 64) - 1, stream())
        np.testing.assert_array_equal(host(o), want)


@pytest.mark.parametrize("d,N", [(64, 1), (64, 2), (64, 333), (64, 8191), (64, 8192), (64, 40001), (16, 1000), (32, 77)])
def test_level_fold_matches_oracle(cuda, d, N):
    """One-pass h(1)/h(2) folds of a dense level vs the reference algebra
    (verify.py:220-230 + gates.py:100-106) restated with oracle/gr.py."""
    from oracle import gr as ogr
    from paper_2411_09287_b200 import grvec, host, _lib
    from paper_2411_09287_b200.rings import modulus_for_degree
    mod = modulus_for_degree(d)
    rng = np.random.default_rng(N + d)
    arrs = [_rand(rng, (N, d)) for _ in range(4)]
    xa, xb, ya, yb = arrs
    pad = lambda a: np.concatenate([a, np.zeros((1, d), np.uint64)]) if N % 2 else a
    with np.errstate(over="ignore"):
        o = lambda a: pad(a)[1::2]
        e = lambda a: pad(a)[0::2]
        two = lambda a: 2 * o(a) - e(a)
        dot = lambda f, g: ogr.dot(f, g, 64, d)
        for role in (0, 1, 2):
            if role == 0:
                w1, w2 = dot(o(xa), o(ya)), dot(two(xa), two(ya))
            elif role == 1:
                w1 = 0 - dot(o(xa), o(yb)) - dot(o(xb), o(ya))
                w2 = 0 - dot(two(xa), two(yb)) - dot(two(xb), two(ya))
            else:
                w1 = dot(o(xa), o(ya) - o(yb)) - dot(o(xb), o(ya))
                w2 = dot(two(xa), two(ya) - two(yb)) - dot(two(xb), two(ya))
            D = [grvec.dev(a) for a in arrs]
            acc = grvec.zeros((2, 2 * d - 1))
            _lib.call("r3_vfy_level_fold", role, D[0].data_ptr(), D[1].data_ptr() if role else None,
                      D[2].data_ptr(), D[3].data_ptr() if role else None, N, d,
                      acc[0].data_ptr(), acc[1].data_ptr(), _lib.stream())
            g1 = host(grvec.reduce_poly(acc[0], mod, 64))
            g2 = host(grvec.reduce_poly(acc[1], mod, 64))
            np.testing.assert_array_equal(g1, w1 & np.uint64(2**64 - 1), err_msg=f"h1 role {role}")
            np.testing.assert_array_equal(g2, w2, err_msg=f"h2 role {role}")


@pytest.mark.parametrize("N", [2 * 16384 * 148 + 4097, (1 << 21) + 1])
def test_level_fold_tc_matches_cuda_core_at_scale(cuda, N):
    """d = 64 tensor-core level fold (lf_tc.cu: o (x) o and t (x) t limb
    products, multi-chunk items whose 2-stage raw / 3-stage limb rings wrap
    many times, odd N) equals the CUDA-core fold (pinned to the oracle
    above) at level-3 sizes.  The folds are sums over row pairs, so the
    CUDA-core side runs over 8190-row slices (4095 pairs each: below the
    tensor-core threshold) accumulating into one output."""
    import torch
    from paper_2411_09287_b200 import grvec, _lib
    g = torch.Generator(device="cuda").manual_seed(N)
    V = [torch.randint(-2**62, 2**62, (N, 64), dtype=torch.int64, device="cuda", generator=g) for _ in range(4)]
    S = 8190

    def fold(role, r0, r1, acc):
        ops = [v[r0:r1] for v in V]
        _lib.call("r3_vfy_level_fold", role, ops[0].data_ptr(), ops[1].data_ptr() if role else None,
                  ops[2].data_ptr(), ops[3].data_ptr() if role else None, r1 - r0, 64,
                  acc[0].data_ptr(), acc[1].data_ptr(), _lib.stream())

    for role in (0, 1, 2):
        tc = grvec.zeros((2, 127))
        fold(role, 0, N, tc)
        cc = grvec.zeros((2, 127))
        for r0 in range(0, N, S):
            fold(role, r0, min(N, r0 + S), cc)
        assert torch.equal(tc, cc), f"role {role}"


@pytest.mark.parametrize("M,K,N", [(128, 32, 64), (256, 96, 128), (384, 4096, 192)])
def test_u64_gemm_tc_exact(cuda, M, K, N):
    """Byte-limb tcgen05 GEMM is exact mod 2^64 (incl. K-concatenation,
    linear-combination operands and addend +/-)."""
    from paper_2411_09287_b200 import grvec, host
    rng = np.random.default_rng(M + K + N)
    X = _rand(rng, (M, K))
    Y = _rand(rng, (M, K))
    W = _rand(rng, (K, N))
    V = _rand(rng, (K, N))
    Z = _rand(rng, (M, N))
    Xd, Yd, Wd, Vd, Zd = (grvec.dev(a) for a in (X, Y, W, V, Z))
    with np.errstate(over="ignore"):
        want = X @ W
        got = host(grvec.u64_gemm([(grvec.limb_tiles_a(Xd), grvec.limb_tiles_b(Wd), K)], M, N))
        np.testing.assert_array_equal(got, want)
        # Z - [X | Y - X] . [W ; V + 3W]
        want2 = Z - (X @ W + (Y - X) @ (V + np.uint64(3) * W))
        pairs = [(grvec.limb_tiles_a(Xd), grvec.limb_tiles_b(Wd), K),
                 (grvec.limb_tiles_a(Yd, 1, Xd, -1), grvec.limb_tiles_b(Vd, 1, Wd, 3), K)]
        got2 = host(grvec.u64_gemm(pairs, M, N, addend=Zd, sub=True))
        np.testing.assert_array_equal(got2, want2)


@pytest.mark.parametrize("d,N", [(64, 4096 + 37), (16, 3001), (8, 515), (32, 128)])
def test_base_fold_matches_definitions(cuda, d, N):
    """r3_vfy_base_fold (one pass over the power table) against the level-1
    folds, level-2 accumulators and z power sum written out from their
    definitions (verify.py:168-179 + 215-241), per role's leg terms."""
    import ctypes as C
    from paper_2411_09287_b200 import grvec, host, _lib
    rng = np.random.default_rng(N * 7 + d)
    pw = _rand(rng, (N, d))
    M = np.uint64(2**64 - 1)
    for role, terms in ((0, [(1, 0, 0)]), (1, [(-1, 0, 1), (-1, 1, 0)]),
                        (2, [(1, 0, 0), (-1, 0, 1), (-1, 1, 0)])):
        comps_x = [_rand(rng, (N,)) for _ in range(2)]
        comps_y = [_rand(rng, (N,)) for _ in range(2)]
        zc = [_rand(rng, (N,)) for _ in range(1 if role == 0 else 2)]
        with np.errstate(over="ignore"):
            pad = lambda a: np.concatenate([a, np.zeros(((-N) % 4,) + a.shape[1:], np.uint64)])
            P = pad(pw)
            X = [pad(a) for a in comps_x]
            Y = [pad(a) for a in comps_y]
            acc = np.zeros((16, d), np.uint64)
            for a in range(4):
                for b in range(4):
                    sab = np.zeros(len(P) // 4, np.uint64)
                    for cf, xi, yi in terms:
                        sab += np.uint64(cf % 2**64) * X[xi][a::4] * Y[yi][b::4]
                    acc[a * 4 + b] = (sab[:, None] * P[a::4]).sum(axis=0)
            # level 1 by definition: pairs (2q, 2q+1), g2 = 2 y_o - y_e
            h1 = np.zeros(d, np.uint64)
            h2 = np.zeros(d, np.uint64)
            for cf, xi, yi in terms:
                c = np.uint64(cf % 2**64)
                xe, xo = X[xi][0::2], X[xi][1::2]
                ye, yo = Y[yi][0::2], Y[yi][1::2]
                g2 = np.uint64(2) * yo - ye
                h1 += ((c * xo * yo)[:, None] * P[1::2]).sum(axis=0)
                h2 += ((c * np.uint64(2) * xo * g2)[:, None] * P[1::2]).sum(axis=0)
                h2 -= ((c * xe * g2)[:, None] * P[0::2]).sum(axis=0)
            zs = [(z[:, None] * pw).sum(axis=0) for z in zc]
        D = lambda a: grvec.dev(a)
        dx, dy, dz, dpw = [D(a) for a in comps_x], [D(a) for a in comps_y], [D(a) for a in zc], D(pw)
        coef = (C.c_int64 * len(terms))(*[t[0] for t in terms])
        xs = (C.c_void_p * len(terms))(*[dx[t[1]].data_ptr() for t in terms])
        ys = (C.c_void_p * len(terms))(*[dy[t[2]].data_ptr() for t in terms])
        zp = (C.c_void_p * len(dz))(*[t.data_ptr() for t in dz])
        g_acc, g_h1, g_h2 = grvec.zeros((16, d)), grvec.zeros((1, d)), grvec.zeros((1, d))
        g_z = grvec.zeros((len(dz), 1, d))
        _lib.call("r3_vfy_base_fold", len(terms), C.addressof(coef), C.addressof(xs), C.addressof(ys),
                  len(dz), C.addressof(zp), 1, N, dpw.data_ptr(), d, g_acc.data_ptr(), g_h1.data_ptr(),
                  g_h2.data_ptr(), g_z.data_ptr(), (1 << 64) - 1, _lib.stream())
        np.testing.assert_array_equal(host(g_acc), acc, err_msg=f"acc role {role}")
        np.testing.assert_array_equal(host(g_h1)[0], h1, err_msg=f"h1 role {role}")
        np.testing.assert_array_equal(host(g_h2)[0], h2, err_msg=f"h2 role {role}")
        for c in range(len(dz)):
            np.testing.assert_array_equal(host(g_z)[c, 0], zs[c], err_msg=f"z{c} role {role}")


def test_staged_input_matches_host_input(cuda):
    """_lib.StagedInput (side-stream H2D started in PRE) gives the same
    shares and opened product as passing the host array."""
    from paper_2411_09287_b200 import gates, host
    from paper_2411_09287_b200._lib import StagedInput
    from paper_2411_09287_b200.runtime import Session
    from paper_2411_09287_b200.sharing import Ring, rec, shc_input_mask, shc_input_online
    from paper_2411_09287_b200.transport import Phase
    rng = np.random.default_rng(3)
    n = 4099
    xh = cuda.from_numpy(rng.integers(0, 2**63, n, dtype=np.int64)).pin_memory()
    yh = cuda.from_numpy(rng.integers(0, 2**63, n, dtype=np.int64)).pin_memory()

    def prog(party, staged):
        ring = Ring(64)
        party.enter_phase(Phase.PRE)
        xs = (StagedInput(xh) if staged else xh) if party.role == 0 else None
        ys = (StagedInput(yh) if staged else yh) if party.role == 1 else None
        xm = shc_input_mask(party, 0, n, ring)
        ym = shc_input_mask(party, 1, n, ring)
        g = gates.mul_prepare(party, xm, ym, n)
        party.round_barrier()
        party.enter_phase(Phase.ONLINE)
        x = shc_input_online(party, 0, xs, xm, n, ring, "x")
        y = shc_input_online(party, 1, ys, ym, n, ring, "y")
        z = gates.mul_finish(party, g, x, y)
        party.enter_phase(Phase.POST)
        party.freeze_logs()
        return host(rec(party, z, "z")), host(z.m) if z.m is not None else None

    a = Session(seed=5).run(prog, True)
    b = Session(seed=5).run(prog, False)
    for r in range(3):
        np.testing.assert_array_equal(a[r][0], b[r][0])
    np.testing.assert_array_equal(a[0][0], xh.numpy().view(np.uint64) * yh.numpy().view(np.uint64))
    np.testing.assert_array_equal(a[1][1], b[1][1])


@pytest.mark.parametrize("N", [2, 3, 1001, 40000, 1 << 18])
def test_level_fold16_tc_matches_cuda_core(cuda, N):
    """r3_vfy_level_fold16_tc (P1's and P2's four leg terms in one
    tensor-core pass) equals the per-role CUDA-core r3_vfy_level_fold on the
    same arrays, incl. odd N (zero odd tail) and a party without terms."""
    import ctypes as C
    import torch
    from paper_2411_09287_b200 import _lib, grvec, host
    d = 16
    rng = np.random.default_rng(N)
    arr = lambda: grvec.dev(_rand(rng, (N, d)))
    m_x, m_y, s1x, s1y, s2x, s2y = (arr() for _ in range(6))

    def core(role, xa, xb, ya, yb):
        acc = torch.zeros((2, 2 * d - 1), dtype=torch.int64, device="cuda")
        _lib.call("r3_vfy_level_fold", role, xa.data_ptr(), xb.data_ptr(), ya.data_ptr(), yb.data_ptr(), N, d,
                  acc[0].data_ptr(), acc[1].data_ptr(), _lib.stream())
        return host(acc)

    want1 = core(1, m_x, s1x, m_y, s1y)
    want2 = core(2, m_x, s2x, m_y, s2y)
    accs = {r: torch.full((2, 2 * d - 1), 7, dtype=torch.int64, device="cuda") for r in (1, 2)}
    terms = [(1, m_x, s1y, None, -1, 0), (1, s1x, m_y, None, -1, 0),
             (2, m_x, m_y, s2y, 1, -1), (2, s2x, m_y, None, -1, 0)]
    P = C.c_void_p
    _lib.call("r3_vfy_level_fold16_tc", 4, (C.c_int * 4)(*[t[0] for t in terms]),
              (P * 4)(*[t[1].data_ptr() for t in terms]), (P * 4)(*[t[2].data_ptr() for t in terms]),
              (P * 4)(*[None if t[3] is None else t[3].data_ptr() for t in terms]),
              (C.c_int64 * 4)(*[t[4] for t in terms]), (C.c_int64 * 4)(*[t[5] for t in terms]), N,
              (P * 3)(None, accs[1][0].data_ptr(), accs[2][0].data_ptr()),
              (P * 3)(None, accs[1][1].data_ptr(), accs[2][1].data_ptr()), _lib.stream())
    np.testing.assert_array_equal(host(accs[1]), want1)
    np.testing.assert_array_equal(host(accs[2]), want2)
    # P0's single term (one item per chunk)
    acc0 = torch.full((2, 2 * d - 1), 5, dtype=torch.int64, device="cuda")
    _lib.call("r3_vfy_level_fold16_tc", 1, (C.c_int * 1)(0), (P * 1)(s1x.data_ptr()), (P * 1)(s2y.data_ptr()),
              (P * 1)(None), (C.c_int64 * 1)(1), (C.c_int64 * 1)(0), N,
              (P * 3)(acc0[0].data_ptr(), None, None), (P * 3)(acc0[1].data_ptr(), None, None), _lib.stream())
    acc_core = torch.zeros((2, 2 * d - 1), dtype=torch.int64, device="cuda")
    _lib.call("r3_vfy_level_fold", 0, s1x.data_ptr(), None, s2y.data_ptr(), None, N, d,
              acc_core[0].data_ptr(), acc_core[1].data_ptr(), _lib.stream())
    np.testing.assert_array_equal(host(acc0), host(acc_core))


@pytest.mark.parametrize("N", [(1 << 16) + 37, 1 << 20])
@pytest.mark.parametrize("joint", [True, False])
@pytest.mark.parametrize("B,d", [(4, 64), (8, 64), (16, 64), (8, 16), (16, 16)])
def test_base_fold_q4_tensor_core_matches_definitions(cuda, N, joint, B, d):
    """r3_vfy_base_fold_q4 on the tensor cores (bf_tc.cu, d = 64) -- the
    headline's base fold -- against its definition
        acc'[a*4+b] = sum_j s^{ab}_j pw4[j],  zraw[c*4+a] = sum_j z_c[4j+a] pw4[j]
    with s^{ab}_j = sum_t coef_t x_t[4j+a] y_t[4j+b] (verify.py:168-179 +
    215-241 restated per block of four).  At these sizes every CTA of the
    persistent grid runs >= 4 (2^16 + 37) and 56 (2^20) 32-block K-steps, so
    the 3-stage TMA / mbarrier ring wraps many times; N = 2^16 + 37 also has
    a ragged last block.  joint=True is the honest-session form (all three
    parties' features in one pass), joint=False one launch per party.
    B = 8 is r3_vfy_base_fold_q8 (blocks of eight against r^(8j): the 64
    accumulators of the first three reductions; one work item per party and
    K-chunk), B = 16 r3_vfy_base_fold_q16 (256 accumulators, three feature
    groups per party and K-chunk); d = 16 runs the same kernels with
    16-coefficient table rows (B operand of 16 columns per limb plane)."""
    import ctypes as C
    from paper_2411_09287_b200 import grvec, host, _lib
    rng = np.random.default_rng(N + 3)
    nblk = (N + B - 1) // B
    pw4 = _rand(rng, (nblk, d))
    roles = {0: [(1, 0, 0)], 1: [(-1, 0, 1), (-1, 1, 0)], 2: [(1, 0, 0), (-1, 0, 1), (-1, 1, 0)]}
    data, want = {}, {}
    for role, terms in roles.items():
        xs = [_rand(rng, (N,)) for _ in range(2)]
        ys = [_rand(rng, (N,)) for _ in range(2)]
        zs = [_rand(rng, (N,)) for _ in range(1 if role == 0 else 2)]
        data[role] = (terms, xs, ys, zs)
        pad = lambda a: np.concatenate([a, np.zeros((-N) % B, np.uint64)]).reshape(nblk, B)
        X, Y, Z = [pad(a) for a in xs], [pad(a) for a in ys], [pad(a) for a in zs]
        with np.errstate(over="ignore"):
            S = np.zeros((nblk, B * B), np.uint64)
            for cf, xi, yi in terms:
                S += np.uint64(cf % 2**64) * (X[xi][:, :, None] * Y[yi][:, None, :]).reshape(nblk, B * B)
            acc = S.T @ pw4
            zr = np.concatenate([z.T @ pw4 for z in Z]) if Z else np.zeros((B, d), np.uint64)
        want[role] = (acc, zr)
    D = grvec.dev
    dev = {r: ([D(a) for a in v[1]], [D(a) for a in v[2]], [D(a) for a in v[3]]) for r, v in data.items()}
    dpw4 = D(pw4)

    def launch(rs):
        P = C.c_void_p
        n = len(rs)
        nterms = (C.c_int * n)(*[len(roles[r]) for r in rs])
        nz = (C.c_int * n)(*[len(dev[r][2]) for r in rs])
        coef = (C.c_int64 * (3 * n))()
        xs, ys, zp = (P * (3 * n))(), (P * (3 * n))(), (P * (2 * n))()
        outs = {}
        for q, r in enumerate(rs):
            for t, (cf, xi, yi) in enumerate(roles[r]):
                coef[3 * q + t], xs[3 * q + t], ys[3 * q + t] = cf, dev[r][0][xi].data_ptr(), dev[r][1][yi].data_ptr()
            for c, zt in enumerate(dev[r][2]):
                zp[2 * q + c] = zt.data_ptr()
            # garbage-filled outputs: the entry point must initialise them
            outs[r] = (grvec.dev(np.full((B * B, d), 0xDEADBEEF, np.uint64)),
                       grvec.dev(np.full((B * len(dev[r][2]), d), 0xDEADBEEF, np.uint64)))
        zstr = (C.c_int64 * n)(*([1] * n))
        acc = (P * n)(*[outs[r][0].data_ptr() for r in rs])
        zr = (P * n)(*[outs[r][1].data_ptr() for r in rs])
        _lib.call(f"r3_vfy_base_fold_q{B}", n, C.addressof(nterms), C.addressof(coef), C.addressof(xs),
                  C.addressof(ys), C.addressof(nz), C.addressof(zp), C.addressof(zstr), N, dpw4.data_ptr(), d,
                  C.addressof(acc), C.addressof(zr), _lib.stream())
        return outs

    outs = launch([0, 1, 2]) if joint else {r: launch([r])[r] for r in roles}
    for r in roles:
        np.testing.assert_array_equal(host(outs[r][0]), want[r][0], err_msg=f"acc role {r}")
        np.testing.assert_array_equal(host(outs[r][1]), want[r][1], err_msg=f"zraw role {r}")


@pytest.mark.parametrize("width", [64, 1])
def test_gr_quad_matches_step_by_step(cuda, width):
    """r3_gr_quad (one launch) equals the reference-shaped helper chain it
    replaces: gr_quad_coeffs (Lagrange weights at an even point), 1 - ze and
    the multiplication matrices of 1 - ze and ze, for every degree."""
    from paper_2411_09287_b200 import grvec, host
    from paper_2411_09287_b200.rings import modulus_for_degree
    rng = np.random.default_rng(width)
    for d in (1, 2, 4, 8, 16, 32, 64):
        mod = modulus_for_degree(d)
        z = rng.integers(0, 2**64, (1, d), dtype=np.uint64) & np.uint64((1 << width) - 1)
        ze = grvec.dev((z * np.uint64(2)) & np.uint64((2**64 - 1) if width == 64 else 1))
        l0, l1, l2 = grvec.gr_quad_coeffs(ze, width, mod)
        (w0, w1, w2), one_m, mats = grvec.gr_quad(ze, width, mod, mats=True)
        np.testing.assert_array_equal(host(w0), host(l0), err_msg=f"l0 d={d}")
        np.testing.assert_array_equal(host(w1), host(grvec.sub(l1, l0, width)), err_msg=f"l1-l0 d={d}")
        np.testing.assert_array_equal(host(w2), host(l2), err_msg=f"l2 d={d}")
        om = grvec.sub(grvec.gr_const(1, mod, width), ze, width)
        np.testing.assert_array_equal(host(one_m), host(om), err_msg=f"1-ze d={d}")
        np.testing.assert_array_equal(host(mats[0]), host(grvec.gr_mulmat(om, mod)), err_msg=f"M(1-ze) d={d}")
        np.testing.assert_array_equal(host(mats[1]), host(grvec.gr_mulmat(ze, mod)), err_msg=f"M(ze) d={d}")


def test_ew3_matches_two_subtractions(cuda):
    from paper_2411_09287_b200 import grvec, host
    rng = np.random.default_rng(3)
    for n in (1, 64, 4099, 1 << 20):
        a, b, c = (grvec.dev(rng.integers(0, 2**64, n, dtype=np.uint64)) for _ in range(3))
        for w in (64, 1, 37):
            np.testing.assert_array_equal(host(grvec.sub3(a, b, c, w)),
                                          host(grvec.sub(grvec.sub(a, b, w), c, w)))


@pytest.mark.parametrize("d,N", [(16, 1), (16, 7), (16, 1000), (8, 4099), (32, 2051), (16, 100003)])
def test_gfv_packed_boolean_levels_match_oracle(cuda, d, N):
    """The packed GF(2^d) boolean verification kernels (csrc/gf2.cu) against
    the oracle's GR(2, d) arithmetic on (n, d) 0/1 words with the general
    formulas (f2 = 2 f1 - f0, line f0 + (f1 - f0) ze): level-0 folds and z
    power sums from the base bits, the first line evaluation from the base
    bits fused with the level-1 folds, then a packed line evaluation written
    unpacked (verify.py:168-241)."""
    import ctypes as C
    import torch
    from oracle import gr as ogr
    from paper_2411_09287_b200 import _lib, grvec, host
    from paper_2411_09287_b200.rings import modulus_for_degree
    rng = np.random.default_rng(N + d)
    mod = modulus_for_degree(d)
    nc, terms = 2, [(1, 1), (1, 0), (0, 1)]
    X = [rng.integers(0, 2, N, dtype=np.uint64) for _ in range(nc)]
    Y = [rng.integers(0, 2, N, dtype=np.uint64) for _ in range(nc)]
    Z = [rng.integers(0, 2, N, dtype=np.uint64) for _ in range(2)]
    r = rng.integers(0, 2, (1, d), dtype=np.uint64)
    zes = [rng.integers(0, 2, (1, d), dtype=np.uint64) for _ in range(2)]
    pw = ogr.powers(r, N, 1, d)
    xl = [ogr.mul(ogr.embed(x, d), pw, 1, d) for x in X]
    yl = [ogr.embed(y, d) for y in Y]

    def folds(xv, yv):
        n = xv[0].shape[0]
        pad = lambda a: np.vstack([a, np.zeros((1, d), np.uint64)]) if n % 2 else a
        h1 = np.zeros((1, d), np.uint64)
        h2 = np.zeros((1, d), np.uint64)
        for tx, ty in terms:
            fx, fy = pad(xv[tx]), pad(yv[ty])
            f2x = (2 * fx[1::2] - fx[0::2]) & np.uint64(1)
            f2y = (2 * fy[1::2] - fy[0::2]) & np.uint64(1)
            h1 = (h1 + ogr.dot(fx[1::2], fy[1::2], 1, d)) & np.uint64(1)
            h2 = (h2 + ogr.dot(f2x, f2y, 1, d)) & np.uint64(1)
        return np.vstack([h1, h2])

    def line(v, ze):
        v = np.vstack([v, np.zeros((1, d), np.uint64)]) if v.shape[0] % 2 else v
        f0, f1 = v[0::2], v[1::2]
        with np.errstate(over="ignore"):
            return (f0 + ogr.mul(f1 - f0, ze, 1, d)) & np.uint64(1)

    P = C.c_void_p
    dev = lambda a: grvec.dev(np.ascontiguousarray(a))
    Xd, Yd, Zd = [dev(x) for x in X], [dev(y) for y in Y], [dev(z) for z in Z]
    rd, zed = dev(r), [dev(z) for z in zes]
    tx = (C.c_int * 3)(*[t[0] for t in terms])
    ty = (C.c_int * 3)(*[t[1] for t in terms])
    scratch = grvec.zeros((4,))
    f_low = mod.lowterms_mask
    out0 = grvec.empty((4, d))
    _lib.call("r3_gfv_base_fold", nc, (P * nc)(*[t.data_ptr() for t in Xd]), (P * nc)(*[t.data_ptr() for t in Yd]),
              3, tx, ty, 2, (P * 2)(*[t.data_ptr() for t in Zd]), N, rd.data_ptr(), d, f_low, out0.data_ptr(),
              scratch.data_ptr(), _lib.stream())
    want0 = folds(xl, yl)
    zs = [(ogr.dot(ogr.embed(z, d), pw, 1, d)) & np.uint64(1) for z in Z]
    np.testing.assert_array_equal(host(out0), np.vstack([want0] + zs))
    # first line evaluation from the base bits + level-1 folds
    n1 = (N + 1) // 2
    o1 = [torch.empty(n1 + 4, dtype=torch.int32, device="cuda") for _ in range(2 * nc)]
    f1 = grvec.empty((2, d))
    _lib.call("r3_gfv_line", 1, nc, (P * nc)(*[t.data_ptr() for t in Xd]), (P * nc)(*[t.data_ptr() for t in Yd]),
              N, rd.data_ptr(), zed[0].data_ptr(), d, f_low, 0, (P * nc)(*[t.data_ptr() for t in o1[:nc]]),
              (P * nc)(*[t.data_ptr() for t in o1[nc:]]), 3, tx, ty, f1.data_ptr(), scratch.data_ptr(), _lib.stream())
    x1 = [line(v, zes[0]) for v in xl]
    y1 = [line(v, zes[0]) for v in yl]
    pack = lambda a: (a.astype(np.uint64) << np.arange(d, dtype=np.uint64)).sum(axis=1).astype(np.uint64)
    for c in range(nc):
        np.testing.assert_array_equal(o1[c][:n1].cpu().numpy().view(np.uint32).astype(np.uint64), pack(x1[c]))
        np.testing.assert_array_equal(o1[nc + c][:n1].cpu().numpy().view(np.uint32).astype(np.uint64), pack(y1[c]))
    np.testing.assert_array_equal(host(f1), folds(x1, y1))
    # packed line evaluation, unpacked output, no fold
    n2 = (n1 + 1) // 2
    o2 = [grvec.empty((n2, d)) for _ in range(2 * nc)]
    _lib.call("r3_gfv_line", 0, nc, (P * nc)(*[t.data_ptr() for t in o1[:nc]]),
              (P * nc)(*[t.data_ptr() for t in o1[nc:]]), n1, None, zed[1].data_ptr(), d, f_low, 1,
              (P * nc)(*[t.data_ptr() for t in o2[:nc]]), (P * nc)(*[t.data_ptr() for t in o2[nc:]]), 0, None, None,
              None, None, _lib.stream())
    for c in range(nc):
        np.testing.assert_array_equal(host(o2[c]), line(x1[c], zes[1]))
        np.testing.assert_array_equal(host(o2[nc + c]), line(y1[c], zes[1]))


@pytest.mark.parametrize("d,n,L", [(16, 64, 4099), (64, 8, 700), (16, 4, 33)])
def test_dot_log_folds_per_lane_match_definitions(cuda, d, n, L):
    """r3_vfy_l1_fold / r3_vfy_l2_fold on a dot log ((n, L) layout, element i
    at (i % n, i // n), power pw[i // n]) -- the per-lane scalar-sum form --
    against the level-1 folds and 16 level-2 accumulators written out from
    their definitions (verify.py:182-212 consolidation + 215-241)."""
    import ctypes as C
    from paper_2411_09287_b200 import grvec, host, _lib
    rng = np.random.default_rng(n * L + d)
    N = n * L
    pw = _rand(rng, (L, d))
    P = np.repeat(pw, n, axis=0)                      # power of element i
    for role, terms in ((0, [(1, 0, 0)]), (2, [(1, 0, 0), (-1, 0, 1), (-1, 1, 0)])):
        cx = [_rand(rng, (n, L)) for _ in range(2)]
        cy = [_rand(rng, (n, L)) for _ in range(2)]
        flat = lambda a: a.T.reshape(-1)              # consolidated order i = l n + k
        X, Y = [flat(a) for a in cx], [flat(a) for a in cy]
        with np.errstate(over="ignore"):
            acc = np.zeros((16, d), np.uint64)
            for a in range(4):
                for b in range(4):
                    sab = np.zeros(N // 4, np.uint64)
                    for cf, xi, yi in terms:
                        sab += np.uint64(cf % 2**64) * X[xi][a::4] * Y[yi][b::4]
                    acc[a * 4 + b] = (sab[:, None] * P[a::4]).sum(axis=0)
            h1 = np.zeros(d, np.uint64)
            h2 = np.zeros(d, np.uint64)
            for cf, xi, yi in terms:
                c = np.uint64(cf % 2**64)
                xe, xo, ye, yo = X[xi][0::2], X[xi][1::2], Y[yi][0::2], Y[yi][1::2]
                h1 += ((c * xo * yo)[:, None] * P[1::2]).sum(axis=0)
                h2 += ((c * (np.uint64(2) * xo - xe) * (np.uint64(2) * yo - ye))[:, None] * P[0::2]).sum(axis=0)
        dx, dy, dpw = [grvec.dev(a) for a in cx], [grvec.dev(a) for a in cy], grvec.dev(pw)
        coef = (C.c_int64 * len(terms))(*[t[0] for t in terms])
        xs = (C.c_void_p * len(terms))(*[dx[t[1]].data_ptr() for t in terms])
        ys = (C.c_void_p * len(terms))(*[dy[t[2]].data_ptr() for t in terms])
        g_acc, g_h1, g_h2 = grvec.empty((16, d)), grvec.empty((1, d)), grvec.empty((1, d))
        _lib.call("r3_vfy_l2_fold", len(terms), coef, xs, ys, N, n, L, 1, dpw.data_ptr(), d, g_acc.data_ptr(),
                  _lib.stream())
        _lib.call("r3_vfy_l1_fold", len(terms), coef, xs, ys, N, n, L, 1, dpw.data_ptr(), d, g_h1.data_ptr(),
                  g_h2.data_ptr(), (1 << 64) - 1, _lib.stream())
        np.testing.assert_array_equal(host(g_acc), acc, err_msg=f"acc role {role}")
        np.testing.assert_array_equal(host(g_h1)[0], h1, err_msg=f"h1 role {role}")
        np.testing.assert_array_equal(host(g_h2)[0], h2, err_msg=f"h2 role {role}")


@pytest.mark.parametrize("N", [8193, 1 << 16])
def test_level_fold_joint_matches_per_party(cuda, N):
    """r3_vfy_level_fold_joint (the three parties' d = 64 dense folds in one
    tensor-core launch, m shared by P1 and P2) against three per-party
    r3_vfy_level_fold launches (pinned to the oracle above)."""
    import ctypes as C
    from paper_2411_09287_b200 import grvec, host, _lib
    rng = np.random.default_rng(N)
    V = {k: grvec.dev(_rand(rng, (N, 64))) for k in ("tx", "ty", "mx", "my", "s1x", "s1y", "s2x", "s2y")}
    want = grvec.zeros((3, 2, 127))
    args = {0: (V["tx"], None, V["ty"], None), 1: (V["mx"], V["s1x"], V["my"], V["s1y"]),
            2: (V["mx"], V["s2x"], V["my"], V["s2y"])}
    for r, (xa, xb, ya, yb) in args.items():
        p = lambda t: None if t is None else t.data_ptr()
        _lib.call("r3_vfy_level_fold", r, p(xa), p(xb), p(ya), p(yb), N, 64, want[r, 0].data_ptr(),
                  want[r, 1].data_ptr(), _lib.stream())
    got = grvec.dev(np.full((3, 2, 127), 0xABCD, np.uint64))
    P3 = C.c_void_p * 3
    _lib.call("r3_vfy_level_fold_joint", *[V[k].data_ptr() for k in ("tx", "ty", "mx", "my", "s1x", "s1y", "s2x", "s2y")],
              N, P3(*[got[r, 0].data_ptr() for r in range(3)]), P3(*[got[r, 1].data_ptr() for r in range(3)]),
              _lib.stream())
    np.testing.assert_array_equal(host(got), host(want))
