"""Circuit front end without a GPU: the parser's acceptance and error
behaviour (reference tests/test_circuit.py:11-31), the plaintext circuit
oracle pinned against the reference's golden circuit runs, and the CLI paths
that finish before any share exists (parse / config errors)."""

import numpy as np
import pytest

from conftest import load_golden
from oracle.circuit_plain import plain_eval, plain_eval_bounds, ulp_distance
from paper_2411_09287_b200 import circuit
from paper_2411_09287_b200.circuit import CircuitParseError


def test_parse_reports_line_numbers():
    with pytest.raises(CircuitParseError) as ei:
        circuit.parse("INPUT 0 0\nBOGUS 1 0\nOUTPUT 0")
    assert ei.value.lineno == 2 and "unknown op 'BOGUS'" in str(ei.value)
    with pytest.raises(CircuitParseError) as ei:
        circuit.parse("INPUT 0 0\nADD 1 0 9\nOUTPUT 1")
    assert "before definition" in str(ei.value)
    with pytest.raises(CircuitParseError) as ei:
        circuit.parse("INPUT 0 0\nADD 1 0 0")
    assert ei.value.lineno == 0
    with pytest.raises(CircuitParseError):
        circuit.parse("INPUT 0 7\nOUTPUT 0")


@pytest.mark.parametrize("text,lineno,what", [
    ("INPUT 0 0\nDOT 1 2 0 0 0\nOUTPUT 1", 2, "DOT arity mismatch"),
    ("INPUT 0 0\nMAXPOOL 1 3 0 0\nOUTPUT 1", 2, "MAXPOOL arity mismatch"),
    ("INPUT 0 0\nMUL 1 0\nOUTPUT 1", 2, "malformed MUL gate"),
    ("INPUT x 0\nOUTPUT 0", 1, "bad wire id 'x'"),
    ("INPUT 0 0\nSCALE 1 zz 0\nOUTPUT 1", 2, "malformed SCALE gate"),
    ("INPUT 0 0\nTRUNC 1 0\nOUTPUT 1", 2, "malformed TRUNC gate"),
    ("INPUT 0 0\nOUTPUT 3", 2, "before definition"),
])
def test_parse_errors(text, lineno, what):
    with pytest.raises(CircuitParseError) as ei:
        circuit.parse(text)
    assert ei.value.lineno == lineno and what in str(ei.value)


def test_parse_structure_comments_and_literals():
    c = circuit.parse("# header\nINPUT 0 1  # owner P1\n\ninput 1 2\nconst 2 0x10\n"
                      "SCALE 3 -1 2\nDOT 4 2 0 1 2 3\nMAXPOOL 5 3 0 1 4\nTRUNC 6 4 8\nOUTPUT 6\nOUTPUT 5\n")
    assert c.inputs == {0: 1, 1: 2}
    assert c.outputs == [6, 5] and c.n_wires == 7
    ops = [(g.op, g.out, g.args, g.lineno) for g in c.gates]
    assert ops[2] == ("CONST", 2, (16,), 5)
    assert ops[3] == ("SCALE", 3, (-1, 2), 6)
    assert ops[4] == ("DOT", 4, (2, (0, 1, 2, 3)), 7)
    assert ops[5] == ("MAXPOOL", 5, ((0, 1, 4),), 8)
    assert ops[6] == ("TRUNC", 6, (4, 8), 9)


def test_load_file(tmp_path):
    p = tmp_path / "c.txt"
    p.write_text("INPUT 0 0\nINPUT 1 1\nMUL 2 0 1\nOUTPUT 2\n")
    c = circuit.load(str(p))
    assert [g.op for g in c.gates] == ["INPUT", "INPUT", "MUL"] and c.outputs == [2]


def _circ_case(name):
    import programs
    spec = {c[0]: c for c in programs.CASES + programs.TAMPER_CASES}[name]
    text, values = programs.CIRCUITS[spec[2][0]]
    return text, values, spec[4].get("ell", 64)


@pytest.mark.parametrize("name", ["circ_mixed", "circ_add_only_R0", "circ_mixed_ell32",
                                  "circ_trunc_relu_pool", "circ_deferred_d64", "circ_random_a",
                                  "circ_random_b_nocheck"])
def test_plain_oracle_matches_reference_runs(name):
    """The plaintext oracle against the opened outputs of the reference's
    own secure runs (every party opened the same values): exact off the
    truncation lineages, within the propagated bound on them."""
    meta, arrays = load_golden(name)
    text, values, ell = _circ_case(name)
    want, bound = plain_eval_bounds(text, values, ell=ell)
    if "trunc" not in name and "random" not in name and "deferred" not in name:
        assert all(int(b[0]) == 0 for b in bound)
    for role in range(3):
        got = arrays[f"p{role}.outputs"]
        for o, (g, w, b) in enumerate(zip(got, want, bound)):
            assert ulp_distance([int(g)], w, ell) <= int(b[0]), (name, role, o)
    assert all(v for k, v in meta["scalars"].items() if "verdicts" in k)


def test_cli_parse_error_exit(tmp_path):
    from paper_2411_09287_b200 import cli
    p = tmp_path / "bad.txt"
    p.write_text("INPUT 0 0\nWAT 1\n")
    assert cli.main(["simulate", str(p)]) == cli.EXIT_PARSE


def test_cli_config_resolution(tmp_path, monkeypatch):
    from paper_2411_09287_b200 import cli
    cfgp = tmp_path / "cfg"
    cfgp.write_text("d=16  # degree\nR=1\nseed=9\nnetwork=wan\n")
    args = cli.build_parser().parse_args(["--config", str(cfgp), "simulate", "c.txt", "--d", "32"])
    cli.resolve(args, cli.read_config(str(cfgp)))
    assert (args.d, args.R, args.seed, args.network, args.ell) == (32, 1, 9, "wan", 64)
    monkeypatch.setenv("RING3PC_SEED", "0x10")
    args = cli.build_parser().parse_args(["soundness"])
    cli.resolve(args, {})
    assert (args.seed, args.gates, args.trials, args.error_site, args.R) == (16, 64, 1000, "gamma", None)
    bad = tmp_path / "bad"
    bad.write_text("novalue\n")
    assert cli.main(["--config", str(bad), "simulate", "c.txt"]) == cli.EXIT_CONFIG


def test_plain_oracle_lanes_and_trunc_sign():
    outs, bound = plain_eval_bounds("INPUT 0 0\nCONST 1 3\nMUL 2 0 1\nTRUNC 3 2 1\nRELU 4 3\nMAXPOOL 5 2 3 1\n"
                      "OUTPUT 3\nOUTPUT 4\nOUTPUT 5", {0: [5, (-5) % 2 ** 64, 0]}, lanes=3)
    m = 2 ** 64
    assert list(outs[0]) == [7, (-8) % m, 0]
    assert list(outs[1]) == [7, 0, 0]
    assert list(outs[2]) == [7, 3, 3]
    assert np.all(outs[0] >= 0)
    assert [list(b) for b in bound] == [[1, 1, 1]] * 3
    _, bound = plain_eval_bounds("INPUT 0 0\nMUL 1 0 0\nTRUNC 2 1 4\nSCALE 3 -3 2\nMUL 4 3 0\nOUTPUT 4",
                                 {0: 100})
    assert int(bound[0][0]) == 3 * 100       # |c| e_trunc, times |x| in the product
