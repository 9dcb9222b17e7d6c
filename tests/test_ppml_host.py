"""Host-side PPML logic (no GPU): fixed-point codec, model chain, fixture
I/O, patch / pool index maps (ppml.py:28-180, 243-273, 437-451 restated as
plain loops here)."""

import numpy as np
import pytest

from paper_2411_09287_b200 import ppml
from paper_2411_09287_b200.rings import ConfigError


def _conv_indices_loops(shape, p):
    c, h, w = shape
    oh = (h + 2 * p["pad"] - p["kh"]) // p["sh"] + 1
    ow = (w + 2 * p["pad"] - p["kw"]) // p["sw"] + 1
    idx = np.full((c * p["kh"] * p["kw"], oh * ow), c * h * w, dtype=np.int64)
    col = 0
    for oy in range(oh):
        for ox in range(ow):
            row = 0
            for ci in range(c):
                for ky in range(p["kh"]):
                    for kx in range(p["kw"]):
                        iy, ix = oy * p["sh"] + ky - p["pad"], ox * p["sw"] + kx - p["pad"]
                        if 0 <= iy < h and 0 <= ix < w:
                            idx[row, col] = (ci * h + iy) * w + ix
                        row += 1
            col += 1
    return idx


@pytest.mark.parametrize("shape,p", [
    ((1, 28, 28), dict(out=5, kh=5, kw=5, sh=2, sw=2, pad=1)),
    ((1, 28, 28), dict(out=6, kh=5, kw=5, sh=1, sw=1, pad=2)),
    ((6, 14, 14), dict(out=16, kh=5, kw=5, sh=1, sw=1, pad=0)),
    ((3, 7, 5), dict(out=2, kh=3, kw=2, sh=2, sw=1, pad=1)),
])
def test_conv_indices_match_loop_form(shape, p):
    np.testing.assert_array_equal(ppml.conv_indices(shape, p), _conv_indices_loops(shape, p))


def test_pool_indices_loop_form():
    c, h, w, win = 3, 4, 6, 2
    got = ppml._pool_indices((c, h, w), win)
    col = 0
    for ci in range(c):
        for oy in range(h // win):
            for ox in range(w // win):
                want = [(ci * h + oy * win + ky) * w + ox * win + kx for ky in range(win) for kx in range(win)]
                assert list(got[:, col]) == want
                col += 1


def test_encode_decode_roundtrip_and_overflow():
    x = np.array([0.0, 1.5, -1.5, 3.25e-3, -7.0, 123.456])
    enc = ppml.encode(x, 16)
    assert enc.dtype == np.uint64
    assert int(enc[2]) == (1 << 64) - 98304
    np.testing.assert_allclose(ppml.decode(enc, 16), np.trunc(x * 2 ** 16) / 2 ** 16)
    with pytest.raises(ConfigError):
        ppml.encode([2.0 ** 47], 16)
    small = ppml.encode([-1.0], 4, ell=16)
    assert int(small[0]) == (1 << 16) - 16
    assert ppml.decode(small, 4, ell=16)[0] == -1.0


def test_model_shapes_and_weight_counts():
    assert ppml.snn_model().shapes() == [(5, 13, 13), (5, 13, 13), (10,)]
    lenet = ppml.lenet28_model()
    assert lenet.shapes()[-1] == (10,) and lenet.shapes()[5] == (16, 5, 5)
    assert [lenet.weight_count(l) for l in lenet.layers if lenet.weight_count(l)] == [150, 2400, 48000, 10080, 840]
    mlp = ppml.secureml_model(np.random.default_rng(0))
    assert [w.size for w in mlp.weights] == [784 * 128, 128 * 128, 1280]
    with pytest.raises(ConfigError):
        ppml.ModelSpec((1, 4, 4), [ppml.Layer("fc", dict(din=15, dout=2))]).shapes()
    with pytest.raises(ConfigError):
        ppml.ModelSpec((1, 5, 5), [ppml.Layer("maxpool", dict(win=2))]).shapes()


def test_model_file_roundtrip(tmp_path):
    m = ppml.snn_model(np.random.default_rng(3))
    path = str(tmp_path / "snn.model")
    ppml.save_model(path, m)
    back = ppml.load_model(path)
    assert back.input_shape == m.input_shape
    assert [(l.kind, l.params) for l in back.layers] == [(l.kind, l.params) for l in m.layers]
    for a, b in zip(back.weights, m.weights):
        np.testing.assert_array_equal(a, b)


def test_lane_split_of_conv_and_fc_batches():
    """verify._FCBatch.split: lane l = a(m) + c(n) for the GEMM-form layers
    (FC lanes m N + n; conv lanes (b, oc, p) at GEMM (b P + p, oc))."""
    from types import SimpleNamespace
    import torch
    from paper_2411_09287_b200.verify import _FCBatch
    z = SimpleNamespace(m=torch.zeros(1), mask=SimpleNamespace(total=torch.zeros(1)))
    M, N = 6, 4
    a, c = _FCBatch.split(SimpleNamespace(M=M, N=N, perm=None, z=z))
    assert (a[:, None] + c[None, :]).reshape(-1).tolist() == list(range(M * N))
    B, out, P = 3, 4, 5                        # conv: M = B P, N = out
    lb, loc, lp = np.meshgrid(np.arange(B), np.arange(out), np.arange(P), indexing="ij")
    perm = torch.as_tensor(((lb * P + lp) * out + loc).reshape(-1))
    a, c = _FCBatch.split(SimpleNamespace(M=B * P, N=out, perm=perm, z=z))
    L = (a[:, None] + c[None, :]).reshape(-1)           # lane of each GEMM index
    assert sorted(L.tolist()) == list(range(B * out * P))
    assert torch.equal(L[perm], torch.arange(B * out * P))
    # a lane order that does not split additively is rejected
    bad = torch.randperm(M * N, generator=torch.Generator().manual_seed(1))
    assert _FCBatch.split(SimpleNamespace(M=M, N=N, perm=bad, z=z)) is None
