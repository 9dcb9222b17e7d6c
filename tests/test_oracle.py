"""Pin the CPU oracle to the live reference's golden vectors (no GPU)."""

import numpy as np
import pytest

from conftest import load_golden


def test_prf_oracle_matches_reference_streams():
    from oracle import prf
    meta, arrays = load_golden("prf")
    for k, spec in enumerate(meta["streams"]):
        s = prf.Stream(bytes.fromhex(spec["seed"]), spec["domain"])
        got = np.concatenate([s.u64(n) for n in spec["draws"]])
        np.testing.assert_array_equal(got, arrays[f"s{k}"])
        # seekable form agrees with the sequential one, including mid-block starts
        key = prf.stream_key(bytes.fromhex(spec["seed"]), spec["domain"])
        np.testing.assert_array_equal(prf.keystream(key, 3, 40), arrays[f"s{k}"][3:43])
    for s, seeds in meta["pair_seeds"].items():
        master = int(s).to_bytes(16, "little")
        assert {k: v.hex() for k, v in prf.pair_seeds(master).items()} == \
            {k: seeds[k] for k in ("01", "02", "12")}
        assert prf.salt(master).hex() == seeds["salt"]


def test_prf_kat():
    from oracle import prf
    s = prf.Stream(bytes(range(16)), "testvec")
    assert s.u64(2).tolist() == [5178918375055795730, 2714498724871165792]


MULV = [("mulv_64_d16_R2", 64, 16, 2, 64, 3), ("mulv_1024_d16_R2", 1024, 16, 2, 64, 11),
        ("mulv_100_d64_R3", 100, 64, 3, 64, 5), ("mulv_1_d16_R0", 1, 16, 0, 64, 6),
        ("mulv_37_d2_R1_ell4", 37, 2, 1, 4, 1), ("mulv_513_d8_R4", 513, 8, 4, 64, 8),
        ("mulv_200_d32_R2", 200, 32, 2, 64, 9), ("mulv_1024_d64_R7", 1024, 64, 7, 64, 11)]


@pytest.mark.parametrize("name,lanes,d,R,ell,seed", MULV)
def test_oracle_mulv_matches_golden(name, lanes, d, R, ell, seed):
    from oracle import mpc
    meta, arrays = load_golden(name)
    res = mpc.mulv(seed=seed, lanes=lanes, d=d, R=R, ell=ell)
    assert res.verdict is True
    assert all(meta["scalars"][f"p{r}.verdict.mul"] for r in range(3))
    for role in range(3):
        for v, nm in ((res.x, "x"), (res.y, "y"), (res.z, "z")):
            for comp, arr in v[role].items():
                np.testing.assert_array_equal(arr, arrays[f"p{role}.{nm}.{comp}"], err_msg=f"{nm} {role} {comp}")
    counters = sorted([[f, t, p, c, n] for (f, t, p, c), n in res.counters.items()])
    assert counters == meta["counters"]
    assert res.sim.rounds == meta["rounds"]
    per = lambda ms: {s: [tuple(m) for m in ms if m[0] == s] for s in range(3)}
    assert per(res.sim.messages) == per(meta["messages"])


def test_oracle_gr_mul_matches_reference_algebra():
    """GR laws the reference tests pin (tests/test_rings.py:55-59)."""
    from oracle import gr
    a = np.array([[3, 1]], dtype=np.uint64)  # ell=4, d=2 hand example: x*x
    x = np.array([[0, 1]], dtype=np.uint64)
    assert gr.mul(x, x, 4, 2).tolist() == [[15, 15]]
    rng = np.random.default_rng(0)
    for d in (2, 4, 8, 16):
        A = rng.integers(0, 2**63, (5, d), dtype=np.uint64)
        B = rng.integers(0, 2**63, (5, d), dtype=np.uint64)
        C = rng.integers(0, 2**63, (5, d), dtype=np.uint64)
        with np.errstate(over="ignore"):
            lhs = gr.mul(A, B + C, 64, d)
            rhs = gr.mul(A, B, 64, d) + gr.mul(A, C, 64, d)
        np.testing.assert_array_equal(lhs, rhs)
        np.testing.assert_array_equal(gr.mul(gr.mul(A, B, 64, d), C, 64, d),
                                      gr.mul(A, gr.mul(B, C, 64, d), 64, d))
    assert a.shape == (1, 2)
