"""uint64 / GR(2^ell, d) array kernels on B200 device tensors.

Drop-in for the reference `ring3pc.grvec` (grvec.py:1-167).  Arrays are
`torch.int64` CUDA tensors carrying uint64 bit patterns: base-ring vectors
(n,) and extension vectors (n, d) with the constant coefficient in column 0
(the reference layout).  Every function launches the hand-written sm_100a
kernels of libr3b200.so (include/r3b200.h); torch is only the allocator,
view/reshape machinery and stream carrier.  `host()` converts to numpy
uint64 for comparison with the reference.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from ._lib import LinOperand, as_i64, call, empty, ptr, stream, to_device, zeros
from .rings import GrModulus, ring_mask

U64 = np.uint64

ADD, SUB, MUL, AND, XOR, OR, RSUB, COPY = range(8)

# rows at which "many elements times one element" switches from the generic
# per-row kernel to the matrix form rows . M_c (tensor-shaped GEMM)
_MATMUL_MIN_ROWS = 64


def umask(width: int) -> np.uint64:
    return U64(ring_mask(width))


def u64(value: int) -> np.uint64:
    return U64(value & ring_mask(64))


def host(t) -> np.ndarray:
    return _lib.to_host(t)


def dev(x) -> torch.Tensor:
    return to_device(x)


def base_from_ints(values, width: int) -> torch.Tensor:
    m = ring_mask(width)
    return to_device(np.array([int(v) & m for v in values], dtype=np.uint64))


def as_gr_rows(rows) -> torch.Tensor:
    return to_device(np.array([[int(c) & ((1 << 64) - 1) for c in r] for r in rows],
                              dtype=np.uint64))


# ---------------------------------------------------------------------------
# elementwise
# ---------------------------------------------------------------------------

def _is_scalar(x) -> bool:
    return not isinstance(x, torch.Tensor) and np.ndim(x) == 0


def _scalar(x) -> int:
    return int(x) & ((1 << 64) - 1)


_M64 = (1 << 64) - 1
_Tensor = torch.Tensor


def ew(op: int, a, b, mask: int) -> torch.Tensor:
    """out = op(a, b) & mask with numpy-style broadcasting (<= 4 dims)."""
    # fast path: contiguous device tensors of one shape, or tensor (op) int
    if type(a) is _Tensor and a.is_cuda and a.is_contiguous():
        tb = type(b)
        if tb is _Tensor:
            if b.shape == a.shape and b.is_contiguous():
                out = torch.empty(a.shape, dtype=torch.int64, device=a.device)
                call("r3_ew_flat", op, a.numel(), out.data_ptr(), a.data_ptr(), b.data_ptr(), 0,
                     mask & _M64, stream())
                return out
        elif tb is int or b is None:
            out = torch.empty(a.shape, dtype=torch.int64, device=a.device)
            call("r3_ew_flat", COPY if b is None else op, a.numel(), out.data_ptr(), a.data_ptr(),
                 None, 0 if b is None else b & _M64, mask & _M64, stream())
            return out
    if _is_scalar(a) and not _is_scalar(b):
        inv = {ADD: ADD, MUL: MUL, AND: AND, XOR: XOR, OR: OR, SUB: RSUB}
        return ew(inv[op], b, a, mask)
    if not isinstance(a, torch.Tensor):
        a = to_device(a)
    if b is not None and not _is_scalar(b) and not isinstance(b, torch.Tensor):
        b = to_device(b)
    if b is None or _is_scalar(b):
        imm = 0 if b is None else _scalar(b)
        shape = tuple(a.shape)
        av = a
        bv = None
    elif a.shape == b.shape:
        shape, av, bv, imm = tuple(a.shape), a, b, 0
    else:
        shape = tuple(torch.broadcast_shapes(a.shape, b.shape))
        av = a.expand(shape)
        bv = b.expand(shape)
        imm = 0
    if len(shape) > 4:
        raise ValueError(f"elementwise kernels take <= 4 dims, got {shape}")
    out = empty(shape)
    nd = len(shape)
    shp = (C.c_int64 * 4)(*shape, *([0] * (4 - nd)))
    ast = (C.c_int64 * 4)(*av.stride(), *([0] * (4 - nd)))
    bst = (C.c_int64 * 4)(*(bv.stride() if bv is not None else [0] * nd), *([0] * (4 - nd)))
    call("r3_ew", op if bv is not None or b is not None else COPY, nd, shp, ptr(out), ptr(av),
         ast, ptr(bv), bst, imm, mask & ((1 << 64) - 1), stream())
    return out


def add(a, b, width: int = 64):
    return ew(ADD, a, b, ring_mask(width))


def sub(a, b, width: int = 64):
    return ew(SUB, a, b, ring_mask(width))


def sub3(a, b, c, width: int = 64):
    """(a - b - c) & mask in one launch for same-shape contiguous device
    tensors (r3_ew3); broadcasting / strided operands take two subtractions."""
    if (type(a) is _Tensor and type(b) is _Tensor and type(c) is _Tensor and a.shape == b.shape == c.shape
            and a.is_contiguous() and b.is_contiguous() and c.is_contiguous() and a.is_cuda):
        out = torch.empty(a.shape, dtype=torch.int64, device=a.device)
        call("r3_ew3", 0, a.numel(), out.data_ptr(), a.data_ptr(), b.data_ptr(), c.data_ptr(),
             ring_mask(width), stream())
        return out
    return sub(sub(a, b, width), c, width)


def mul(a, b, width: int = 64):
    return ew(MUL, a, b, ring_mask(width))


def vmask(a, width: int):
    if width == 64:
        return a
    return ew(AND, a, ring_mask(width), ring_mask(64))


def vneg(a, width: int):
    return ew(RSUB, a, 0, ring_mask(width))


def vscale(a, c: int, width: int):
    return ew(MUL, a, _scalar(c), ring_mask(width))


def arith_rshift(a, t: int, width: int):
    """Arithmetic right shift of width-bit two's-complement patterns."""
    if t == 0:
        return ew(COPY, a, None, ring_mask(64))
    if not 0 < t < width:
        raise ValueError(f"shift {t} out of range for width {width}")
    src = a.contiguous()
    out = empty(src.shape)
    call("r3_ars", ptr(src), src.numel(), t, width, ptr(out), stream())
    return out


def to_signed(a, width: int):
    """Signed interpretation as host int64 (the reference returns int64)."""
    h = host(a).astype(np.int64) if width == 64 else host(a)
    if width == 64:
        return h
    half = 1 << (width - 1)
    v = h.astype(np.int64)
    return np.where(h >= half, v - (1 << width), v)


def bit_planes(a, nbits: int) -> torch.Tensor:
    """(nbits, lanes) of (a >> j) & 1 (nonlinear.py:273)."""
    src = a.contiguous()
    out = empty((nbits, src.shape[0]))
    call("r3_bit_planes", ptr(src), src.shape[0], nbits, ptr(out), stream())
    return out


def count_nonequal(a, b=None, into: torch.Tensor | None = None) -> torch.Tensor:
    """Device scalar #{a != b} (b None: #{a != 0}); accumulates into `into`
    when given (deferred consistency checks)."""
    a = a.contiguous()
    cnt = zeros((1,)) if into is None else into
    if b is not None:
        b = b.contiguous()
        if b.shape != a.shape:
            cnt.add_(1)
            return cnt
    call("r3_count_nonequal", ptr(a), ptr(b), a.numel(), ptr(cnt), stream())
    return cnt


def sum_axis0(a: torch.Tensor, width: int, keepdims: bool = False) -> torch.Tensor:
    """np.add.reduce(a, axis=0) masked to width bits."""
    if a.dim() == 0:
        raise ValueError("sum over a scalar")
    n = a.shape[0]
    rest = tuple(a.shape[1:])
    inner = int(np.prod(rest)) if rest else 1
    src = a.reshape(n, inner)
    if inner > 1 and src.stride(1) != 1:
        src = src.contiguous()
    rs = src.stride(0) if n > 1 else inner
    out = empty((inner,))
    call("r3_sum_axis0", ptr(src), n, inner, rs, ptr(out), ring_mask(width), 0, stream())
    shape = ((1,) if keepdims else ()) + rest
    return out.reshape(shape)


# ---------------------------------------------------------------------------
# GR(2^ell, d)
# ---------------------------------------------------------------------------

def gr_embed(base, mod: GrModulus) -> torch.Tensor:
    """(n,) base values -> (n, d), constant coefficient set."""
    base = base if isinstance(base, torch.Tensor) else to_device(base)
    out = zeros(tuple(base.shape) + (mod.degree,))
    out[..., 0] = base
    return out


_CONSTS: dict = {}


def gr_const(value: int, mod: GrModulus, width: int) -> torch.Tensor:
    """(1, d) embedded constant.  Built once per device on the host side and
    reused: writing a python scalar into a device tensor would be a blocking
    host->device copy on the hot path (tensors are never mutated in place)."""
    key = (value & ring_mask(width), mod.degree, torch._C._cuda_getDevice())
    t = _CONSTS.get(key)
    if t is None:
        host_v = np.zeros((1, mod.degree), dtype=np.uint64)
        host_v[0, 0] = key[0]
        t = _CONSTS[key] = to_device(host_v)
    return t


def lin(*terms, nvalid=None) -> LinOperand:
    """LinOperand from (coef, tensor2d) pairs; each tensor (rows, d) with
    unit coefficient stride (row stride may be anything, 0 = broadcast)."""
    op = LinOperand()
    op.nterms = len(terms)
    for q, (coef, t) in enumerate(terms):
        if t.dim() != 2 or (t.shape[1] > 1 and t.stride(1) != 1):
            raise ValueError("lin operand wants (rows, d) with contiguous coefficients")
        op.p[q] = ptr(t)
        op.rowstride[q] = t.stride(0) if t.shape[0] > 1 else 0
        op.nvalid[q] = (1 << 62) if (nvalid is None or nvalid[q] is None) else nvalid[q]
        op.coef[q] = _scalar(coef)
    for q in range(len(terms), 4):
        op.p[q] = None
        op.rowstride[q] = 0
        op.nvalid[q] = 0
        op.coef[q] = 0
    return op


def _rows2d(t: torch.Tensor, d: int) -> torch.Tensor:
    if t.dim() != 2 or t.shape[-1] != d:
        raise ValueError("coefficient count does not match modulus degree")
    if d > 1 and t.stride(1) != 1:
        t = t.contiguous()
    return t


def gr_mulmat(c: torch.Tensor, mod: GrModulus) -> torch.Tensor:
    """(d, d) matrix M with (a * c) = a . M."""
    d = mod.degree
    c = c.reshape(-1, d)[0].contiguous()
    M = empty((d, d))
    call("r3_gr_mulmat", ptr(c), d, mod.lowterms_mask, ptr(M), stream())
    return M


def gr_matmul(A: LinOperand, M: torch.Tensor, rows: int, d: int, width: int,
              C_add: LinOperand | None = None, out: torch.Tensor | None = None):
    if out is None:
        out = empty((rows, d))
    call("r3_gr_matmul", A, ptr(M), 1 if C_add is not None else 0,
         C_add if C_add is not None else LinOperand(), ptr(out), rows, d, ring_mask(width),
         stream())
    return out


def gr_mul(a, b, width: int, mod: GrModulus) -> torch.Tensor:
    """Product in GR(2^width, d) mod f, rows broadcast on axis 0."""
    d = mod.degree
    a = a if isinstance(a, torch.Tensor) else to_device(a)
    b = b if isinstance(b, torch.Tensor) else to_device(b)
    if a.shape[-1] != d or b.shape[-1] != d:
        raise ValueError("coefficient count does not match modulus degree")
    if d == 1:
        return ew(MUL, a, b, ring_mask(width))
    a, b = _rows2d(a, d), _rows2d(b, d)
    n = max(a.shape[0], b.shape[0])
    if a.shape[0] not in (1, n) or b.shape[0] not in (1, n):
        raise ValueError(f"cannot broadcast {tuple(a.shape)} with {tuple(b.shape)}")
    a_one = a.shape[0] == 1 or a.stride(0) == 0
    b_one = b.shape[0] == 1 or b.stride(0) == 0
    if d >= 8 and n >= _MATMUL_MIN_ROWS and a_one != b_one:
        one, many = (a, b) if a_one else (b, a)
        M = gr_mulmat(one[:1], mod)
        return rows_times(many, M, n, width)
    out = empty((n, d))
    a_rs = 0 if a_one else a.stride(0)
    b_rs = 0 if b_one else b.stride(0)
    call("r3_gr_mul", ptr(a), a_rs, ptr(b), b_rs, ptr(out), n, d, mod.lowterms_mask,
         ring_mask(width), stream())
    return out


def gr_scale_rows(s: torch.Tensor, g: torch.Tensor, width: int) -> torch.Tensor:
    """out[i] = s[i] * g[i] for base scalars s (n,) and GR rows g (n|1, d)."""
    d = g.shape[-1]
    g = _rows2d(g, d)
    n = max(s.shape[0], g.shape[0])
    out = empty((n, d))
    s_st = 0 if s.shape[0] == 1 else s.stride(0)
    g_rs = 0 if g.shape[0] == 1 else g.stride(0)
    call("r3_gr_scale_rows", ptr(s), s_st, ptr(g), g_rs, ptr(out), n, d, ring_mask(width),
         stream())
    return out


def _mul_gf2_packed(a, b, mod):  # pragma: no cover - parity alias
    return gr_mul(a, b, 1, mod)


def gr_scale_base(a, c, width: int):
    """Coefficient-wise product with base scalars c of shape (n,) or ()."""
    if _is_scalar(c):
        return ew(MUL, a, _scalar(c), ring_mask(width))
    c = c if isinstance(c, torch.Tensor) else to_device(c)
    return ew(MUL, a, c[..., None], ring_mask(width))


def dotsum_acc(d: int) -> torch.Tensor:
    return zeros((2 * d - 1,))


def dotsum_add(acc: torch.Tensor, F: LinOperand, G: LinOperand, rows: int, d: int) -> None:
    call("r3_gr_dotsum", F, G, rows, d, ptr(acc), stream())


def reduce_poly(acc: torch.Tensor, mod: GrModulus, width: int, out: torch.Tensor | None = None,
                accumulate: bool = False) -> torch.Tensor:
    d = mod.degree
    if out is None:
        out = empty((1, d))
    call("r3_gr_reduce_poly", ptr(acc), d, mod.lowterms_mask, ptr(out), ring_mask(width),
         1 if accumulate else 0, stream())
    return out


def reduce_poly_rows(acc: torch.Tensor, mod: GrModulus, width: int) -> torch.Tensor:
    """Every (2d - 1)-word row of the contiguous acc reduced: (rows, d), one
    launch (r3_gr_reduce_poly_rows)."""
    d = mod.degree
    rows = acc.numel() // (2 * d - 1)
    out = empty((rows, d))
    call("r3_gr_reduce_poly_rows", ptr(acc), rows, d, mod.lowterms_mask, ptr(out), ring_mask(width), stream())
    return out


def gr_dot(a, b, width: int, mod: GrModulus) -> torch.Tensor:
    """Sum of pairwise products, shape (1, d)."""
    d = mod.degree
    a, b = _rows2d(a, d), _rows2d(b, d)
    n = max(a.shape[0], b.shape[0])
    acc = dotsum_acc(d)
    dotsum_add(acc, lin((1, a)), lin((1, b)), n, d)
    return reduce_poly(acc, mod, width)


def gr_powers(r, n: int, width: int, mod: GrModulus) -> torch.Tensor:
    """(n, d) array r^0 .. r^(n-1) by block doubling (grvec.py:130-141):
    each doubling round is one rows . M_step matrix product."""
    d = mod.degree
    r = r.reshape(1, d)
    out = empty((n, d))          # every row is written by the doubling rounds
    if n == 0:
        return out
    out[0:1] = gr_const(1, mod, width)
    filled = 1
    while filled < n:
        take = min(filled, n - filled)
        step = gr_mul(out[filled - 1:filled], r, width, mod)
        if d >= 8:
            M = gr_mulmat(step, mod)
            rows_times(out[:take], M, take, width, out=out[filled:filled + take])
        else:
            out[filled:filled + take] = gr_mul(out[:take], step, width, mod)
        filled += take
    return out


def gr_line_eval(p0, p1, z, width: int, mod: GrModulus):
    """z*p1 - (z-1)*p0, rows of p0/p1; z shaped (1, d)."""
    one = gr_const(1, mod, width)
    zm1 = sub(z, one, width)
    return sub(gr_mul(z, p1, width, mod), gr_mul(zm1, p0, width, mod), width)


def _check_even(z_even) -> None:
    if int(count_nonequal(ew(AND, z_even, 1, ring_mask(64))).item()):
        raise ValueError("even evaluation point required")


def gr_quad_coeffs(z_even, width: int, mod: GrModulus, check: bool = True):
    """Lagrange weights (l0, l1, l2) at an even point, each (1, d)."""
    if check:
        _check_even(z_even)
    u = _shr1(z_even)
    one = gr_const(1, mod, width)
    two = gr_const(2, mod, width)
    l0 = gr_mul(sub(z_even, one, width), sub(u, one, width), width, mod)
    l1 = gr_mul(z_even, sub(two, z_even, width), width, mod)
    l2 = gr_mul(u, sub(z_even, one, width), width, mod)
    return l0, l1, l2


def gr_quad(z_even, width: int, mod: GrModulus, mats: bool = True, check: bool = True):
    """((l0, l1 - l0, l2), 1 - z, (M(1 - z), M(z)) or None) in one launch
    (r3_gr_quad): gr_quad_coeffs plus the line-evaluation operands."""
    if check:
        _check_even(z_even)
    d = mod.degree
    out = empty((4, d))
    Mo = empty((d, d)) if mats else None
    Mz = empty((d, d)) if mats else None
    call("r3_gr_quad", ptr(z_even.reshape(-1, d)[0].contiguous()), d, mod.lowterms_mask, ring_mask(width),
         ptr(out), ptr(Mo), ptr(Mz), stream())
    return (out[0:1], out[1:2], out[2:3]), out[3:4], ((Mo, Mz) if mats else None)


def _shr1(a):
    # logical shift right by one: (a >> 1) == arith_rshift(a,1,64) & (2^63-1)
    return ew(AND, arith_rshift(a, 1, 64), (1 << 63) - 1, ring_mask(64))


def gr_quad_eval(h0, h1, h2, z_even, width: int, mod: GrModulus):
    l0, l1, l2 = gr_quad_coeffs(z_even, width, mod)
    out = add(gr_mul(l0, h0, width, mod), gr_mul(l1, h1, width, mod), width)
    return add(out, gr_mul(l2, h2, width, mod), width)


# ---------------------------------------------------------------------------
# many elements times one element: tensor-core dispatch
# ---------------------------------------------------------------------------

def _tc_ok(t: torch.Tensor) -> bool:
    return (t.shape[0] <= 1 or t.stride(0) % 2 == 0) and t.data_ptr() % 16 == 0 and t.stride(-1) == 1


def rows_times(P0: torch.Tensor, M0: torch.Tensor, rows: int, width: int, *,
               P1: torch.Tensor | None = None, M1: torch.Tensor | None = None,
               nvalid=(None, None), out: torch.Tensor | None = None) -> torch.Tensor:
    """out[r] = P0[r] . M0 (+ P1[r] . M1): rows of GR elements times fixed
    elements given by their multiplication matrices.  d = 64 and d = 16 run
    on the tensor cores (r3_gr_matmul2_tc / _tc16, int8 byte limbs); other
    degrees on the CUDA-core matrix kernel.  Rows at or beyond nvalid[q] of P_q are zero."""
    d = M0.shape[0]
    n0 = rows if nvalid[0] is None else nvalid[0]
    n1 = rows if nvalid[1] is None else nvalid[1]
    if out is None:
        out = empty((rows, d))
    if rows == 0:
        return out
    if d in (16, 64) and _tc_ok(P0) and (P1 is None or _tc_ok(P1)):
        fn = "r3_gr_matmul2_tc" if d == 64 else "r3_gr_matmul2_tc16"
        rs0 = P0.stride(0) if P0.shape[0] > 1 else d
        if P1 is not None and P1.shape[0] > 0:
            rs1 = P1.stride(0) if P1.shape[0] > 1 else d
            call(fn, ptr(P0), rs0, n0, ptr(P1), rs1, n1, ptr(M0), ptr(M1),
                 ptr(out), rows, ring_mask(width), stream())
        else:
            call(fn, ptr(P0), rs0, n0, None, 0, 0, ptr(M0), None,
                 ptr(out), rows, ring_mask(width), stream())
        return out
    if P1 is None or P1.shape[0] == 0:
        return gr_matmul(lin((1, P0), nvalid=[n0]), M0, rows, d, width, out=out)
    # CUDA-core form: P0.M0 + P1.M1 with M0 = M(1 - z), M1 = M(z) is
    # P0 + (P1 - P0).M1 when M0 + M1 = I (line evaluation); general case:
    tmp = gr_matmul(lin((1, P1), nvalid=[n1]), M1, rows, d, width)
    return gr_matmul(lin((1, P0), nvalid=[n0]), M0, rows, d, width,
                     C_add=lin((1, tmp)), out=out)


def rows_times2_batch(jobs: list, M0: torch.Tensor, M1: torch.Tensor, width: int) -> list:
    """[rows_times(ev, M0, n0, P1=od, M1=M1, nvalid=(n0, n1)) for (ev, od,
    n0, n1) in jobs]: for d = 64 / 16 every job with both operands present
    runs in ONE tensor-core launch (r3_gr_matmul2_tc_multi / _tc16_multi,
    up to 8 jobs share the B planes of M0 / M1); other shapes one
    rows_times each."""
    d = M0.shape[0]
    outs = [None] * len(jobs)
    batch = []
    for i, (ev, od, n0, n1) in enumerate(jobs):
        if d in (16, 64) and n0 >= 1 and n1 >= 1 and _tc_ok(ev) and _tc_ok(od):
            batch.append(i)
        else:
            outs[i] = rows_times(ev, M0, n0, width, P1=od, M1=M1, nvalid=(n0, n1))
    for s in range(0, len(batch), 8):
        idx = batch[s:s + 8]
        k = len(idx)
        P = C.c_void_p * k
        L = C.c_int64 * k
        for i in idx:
            outs[i] = empty((jobs[i][2], d))
        rs = lambda t: t.stride(0) if t.shape[0] > 1 else d
        call("r3_gr_matmul2_tc_multi" if d == 64 else "r3_gr_matmul2_tc16_multi", k,
             P(*[jobs[i][0].data_ptr() for i in idx]),
             L(*[rs(jobs[i][0]) for i in idx]), L(*[jobs[i][2] for i in idx]),
             P(*[jobs[i][1].data_ptr() for i in idx]), L(*[rs(jobs[i][1]) for i in idx]),
             L(*[jobs[i][3] for i in idx]), ptr(M0), ptr(M1), P(*[outs[i].data_ptr() for i in idx]),
             L(*[jobs[i][2] for i in idx]), ring_mask(width), stream())
    return outs


def rows_times_multi(P: torch.Tensor, Ms: list, rows: int, width: int, outs: list) -> list:
    """outs[k][r] = P[r] . Ms[k] for d = 64 and up to 4 matrices in one pass
    over P (r3_gr_matmul_q_tc); other degrees / layouts one rows_times each."""
    d = Ms[0].shape[0]
    if d == 64 and len(Ms) <= 4 and _tc_ok(P) and all(o.is_contiguous() for o in outs):
        if rows:
            rs = P.stride(0) if P.shape[0] > 1 else d
            pm = (C.c_void_p * len(Ms))(*[m.data_ptr() for m in Ms])
            po = (C.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
            call("r3_gr_matmul_q_tc", ptr(P), rs, rows, pm, po, len(Ms), ring_mask(width), stream())
        return outs
    for M, o in zip(Ms, outs):
        rows_times(P, M, rows, width, out=o)
    return outs


# ---------------------------------------------------------------------------
# u64 GEMM on the tensor cores (share-domain matmul)
# ---------------------------------------------------------------------------

def limb_tiles_a(P0: torch.Tensor, c0: int = 1, P1: torch.Tensor | None = None, c1: int = 0):
    """rows x K operand (c0 P0 + c1 P1) -> UMMA-ready byte-limb tiles."""
    rows, K = P0.shape
    dst = torch.empty(rows * K * 8, dtype=torch.uint8, device=P0.device)
    call("r3_limb_tiles_a", ptr(P0.contiguous()), _scalar(c0),
         ptr(P1.contiguous()) if P1 is not None else None, _scalar(c1), rows, K, ptr(dst), stream())
    return dst


def limb_tiles_b(P0: torch.Tensor, c0: int = 1, P1: torch.Tensor | None = None, c1: int = 0):
    """K x cols operand (c0 P0 + c1 P1) -> K-major byte-limb tiles."""
    K, cols = P0.shape
    dst = torch.empty(K * cols * 8, dtype=torch.uint8, device=P0.device)
    call("r3_limb_tiles_b", ptr(P0.contiguous()), _scalar(c0),
         ptr(P1.contiguous()) if P1 is not None else None, _scalar(c1), K, cols, ptr(dst), stream())
    return dst


def u64_gemm(pairs, M: int, N: int, width: int = 64, addend: torch.Tensor | None = None,
             sub: bool = False) -> torch.Tensor:
    """addend +/- sum_p A_p . B_p over Z_2^width; pairs = [(a_tiles, b_tiles, K)]."""
    out = empty((M, N))
    a = (C.c_void_p * len(pairs))(*[ptr(p[0]) for p in pairs])
    b = (C.c_void_p * len(pairs))(*[ptr(p[1]) for p in pairs])
    k = (C.c_int64 * len(pairs))(*[p[2] for p in pairs])
    call("r3_u64_gemm_tc", len(pairs), a, b, k, M, N,
         ptr(addend.contiguous()) if addend is not None else None, 1 if sub else 0,
         ptr(out), ring_mask(width), stream())
    return out


_PTRS12 = C.c_void_p * 12


def ew_fields(op: int, a: list, b, mask: int) -> list:
    """[op(a_c, b_c) & mask] for up to 4 same-shape contiguous tensors in one
    launch (b: list of tensors, one int for all, or None for a copy).
    Components that do not qualify fall back to one ew call each."""
    k = len(a)
    bl = b if isinstance(b, list) else None
    ok = 0 < k <= 4
    if ok:
        shape = a[0].shape
        for c in range(k):
            t = a[c]
            if type(t) is not _Tensor or t.shape != shape or not t.is_contiguous() or not t.is_cuda:
                ok = False
                break
            if bl is not None:
                u = bl[c]
                if type(u) is not _Tensor or u.shape != shape or not u.is_contiguous():
                    ok = False
                    break
        if ok and bl is None and b is not None and type(b) is not int:
            ok = False
    if not ok:
        return [ew(op, a[c], bl[c] if bl is not None else b, mask) for c in range(k)]
    n = a[0].numel()
    # one allocation for the k outputs (value semantics: the views are never
    # written after this call)
    # rows padded to an even word count keep every output 16-byte aligned
    npad = n + (n & 1)
    block = torch.empty((k, npad), dtype=torch.int64, device=a[0].device)
    outs = [block[c, :n].view(shape) for c in range(k)]
    base_out = block.data_ptr()
    step = npad * 8
    arr = _PTRS12(*[base_out + c * step for c in range(k)], *([None] * (4 - k)),
                  *[t.data_ptr() for t in a], *([None] * (4 - k)),
                  *([u.data_ptr() for u in bl] if bl is not None else [None] * k), *([None] * (4 - k)))
    base = C.addressof(arr)
    call("r3_ew_multi", COPY if b is None else op, k, n, base, base + 32, base + 64 if bl is not None else None,
         0 if (b is None or bl is not None) else b & _M64, mask & _M64, stream())
    return outs


def gr_lincomb(terms: list, coeffs: list, width: int, mod: GrModulus) -> list:
    """[sum_t terms[t][f] * coeffs[t] for each field f] in GR(2^width, d):
    terms[t] is a list of k <= 4 same-shape (rows, d) tensors, coeffs[t] one
    public element; one launch for all fields (r3_gr_lincomb)."""
    d = mod.degree
    nterms, k = len(terms), len(terms[0])
    shape = terms[0][0].shape
    # the kernel reads rows of d words: any contiguous tensor is its own
    # (rows, d) view, so only non-contiguous operands are copied
    flat = [t if t.is_contiguous() else t.contiguous() for row in terms for t in row]
    cs = [(c if c.is_contiguous() else c.contiguous()) if isinstance(c, torch.Tensor)
          else to_device(c).reshape(-1)[:d] for c in coeffs]
    rows = flat[0].numel() // d
    block = torch.empty((k,) + tuple(shape), dtype=torch.int64, device=flat[0].device)
    outs = list(block.unbind(0)) if k > 1 else [block[0]]
    step = rows * d * 8
    pa = (C.c_void_p * (nterms * k))(*[t.data_ptr() for t in flat])
    pc = (C.c_void_p * nterms)(*[c.data_ptr() for c in cs])
    po = (C.c_void_p * k)(*[block.data_ptr() + i * step for i in range(k)])
    call("r3_gr_lincomb", k, nterms, C.addressof(pa), C.addressof(pc), C.addressof(po), rows, d,
         mod.lowterms_mask, ring_mask(width), stream())
    return outs
