"""PRF kernel parity: reference KAT + golden streams + seekable oracle."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def test_prf_golden_streams(cuda):
    from paper_2411_09287_b200 import host
    from paper_2411_09287_b200.prg import Prg
    meta, arrays = load_golden("prf")
    for k, spec in enumerate(meta["streams"]):
        p = Prg(bytes.fromhex(spec["seed"]), spec["domain"])
        got = np.concatenate([host(p.draw_u64(n)) for n in spec["draws"]])
        np.testing.assert_array_equal(got, arrays[f"s{k}"])
    p = Prg(bytes(range(16)), "m")
    np.testing.assert_array_equal(host(p.draw_bits(100)), arrays["bits"])
    np.testing.assert_array_equal(host(p.draw_base(64, 4)), arrays["base4"])


def test_prf_kat(cuda):
    from paper_2411_09287_b200 import host
    from paper_2411_09287_b200.prg import Prg
    p = Prg(bytes(range(16)), "testvec")
    assert host(p.draw_u64(2)).tolist() == [5178918375055795730, 2714498724871165792]


@pytest.mark.parametrize("first,n", [(0, 1), (1, 1), (1, 2), (3, 1000), (12345, 77777),
                                      (2**33 + 1, 4097), (0, 1 << 22), (2**40 + 3, (1 << 18) + 5)])
def test_prf_seek_vs_oracle(cuda, first, n):
    import ctypes as C
    from oracle import prf as oprf
    from paper_2411_09287_b200 import host, _lib
    from paper_2411_09287_b200.prg import round_keys
    key = bytes(range(100, 116))
    out = _lib.empty((n,))
    _lib.call("r3_prf_ctr", round_keys(key), first, n, (1 << 64) - 1, 0, out.data_ptr(), _lib.stream())
    np.testing.assert_array_equal(host(out), oprf.keystream(key, first, n))


@pytest.mark.parametrize("first,lanes", [(0, 1 << 17), (7, (1 << 17) + 3), (2**35, 1 << 16)])
def test_prf_bits_packed_bulk_vs_oracle(cuda, first, lanes):
    """Bulk bit draws (the four-table AES kernel): bit j of lane l is bit 0 of
    stream word first + j * lanes + l, on sampled lanes incl. both ends."""
    from oracle import prf as oprf
    from paper_2411_09287_b200 import host, _lib
    from paper_2411_09287_b200.prg import round_keys
    key = bytes(range(7, 23))
    nbits = 64
    out = _lib.empty((lanes,))
    _lib.call("r3_prf_bits_packed", round_keys(key), first, nbits, lanes, out.data_ptr(), _lib.stream())
    got = host(out)
    rng = np.random.default_rng(lanes)
    for l in [0, 1, lanes - 1] + [int(v) for v in rng.integers(0, lanes, 13)]:
        want = 0
        for j in range(nbits):
            want |= (int(oprf.keystream(key, first + j * lanes + l, 1)[0]) & 1) << j
        assert int(got[l]) == want, l
