"""Circuit evaluator and CLI on the B200 backend (reference
tests/test_circuit.py, tests/test_cli.py, tests/test_acceptance.py:160-208).

The golden circuit runs themselves (shares, transcript, payload hashes) are
checked by test_gpu_golden.py; here: the reference's behavioural tests, the
batched evaluator against the plaintext oracle, and the CLI commands."""

import numpy as np
import pytest

from oracle.circuit_plain import plain_eval_bounds, ulp_distance

pytestmark = pytest.mark.gpu


def _run(prog, *args, seed=0, ell=64, adversary=None):
    from paper_2411_09287_b200.runtime import Session
    sess = Session(seed=seed, ell=ell, adversary=adversary)
    return sess, sess.run(prog, *args)


def test_trunc_requires_mul_or_dot_producer(cuda):
    from paper_2411_09287_b200 import circuit
    circ = circuit.parse("INPUT 0 0\nTRUNC 1 0 4\nOUTPUT 1")
    with pytest.raises(circuit.CircuitParseError):
        _run(circuit.evaluate, circ, {0: 5}, 16, 0, False)


def test_add_only_circuit_zero_online_mul_bytes(cuda):
    from paper_2411_09287_b200 import circuit
    from paper_2411_09287_b200.transport import Phase
    circ = circuit.parse("INPUT 0 0\nINPUT 1 1\nADD 2 0 1\nOUTPUT 2")
    sess, res = _run(circuit.evaluate, circ, {0: 1, 1: 2}, 16, 0)
    assert res[0][0] == [3]
    assert sess.transcript.bytes_sent(phase=Phase.ONLINE) == 24


def test_single_mul_round_count_and_abort(cuda):
    from paper_2411_09287_b200 import circuit
    from paper_2411_09287_b200.transport import AbortError, AdversaryConfig, Phase
    circ = circuit.parse("INPUT 0 0\nINPUT 1 1\nMUL 2 0 1\nOUTPUT 2")
    sess, res = _run(circuit.evaluate, circ, {0: 6, 1: 7}, 16, 2)
    assert res[0][0] == [42] and res[0][1] and all(res[0][1].values())
    assert sess.transcript.rounds[Phase.ONLINE] == 1
    with pytest.raises(AbortError):
        _run(circuit.evaluate, circ, {0: 6, 1: 7}, 16, 2, adversary=AdversaryConfig.parse("P0:gamma:+1"))


def test_random_circuits_quick(cuda):
    """Ten seeded random circuits over every gate kind (tests/programs.py
    random_circuit) opened against the plaintext oracle."""
    import programs
    from paper_2411_09287_b200 import circuit
    for s in range(10):
        text, values = programs.random_circuit(1000 + s, n_gates=10)
        _, res = _run(circuit.evaluate, circuit.parse(text), values, 16, 1, seed=s)
        want, bound = plain_eval_bounds(text, values)
        for g, w, b in zip(res[0][0], want, bound):
            assert ulp_distance([g], w) <= int(b[0]), (s, text)


def test_batch_of_one_is_evaluate(cuda):
    """evaluate_batch at one lane reproduces evaluate: outputs, verdicts and
    the whole message log (same PRF draws, same gates, same order)."""
    import programs
    from paper_2411_09287_b200 import circuit
    text, values = programs.CIRCUITS["random_a"]
    circ = circuit.parse(text)
    s1, r1 = _run(circuit.evaluate, circ, values, 16, 1, seed=4)
    s2, r2 = _run(circuit.evaluate_batch, circ, values, 1, 16, 1, seed=4)
    assert [int(o[0]) for o in r2[0][0]] == r1[0][0] and r2[0][1] == r1[0][1]
    assert s1.transcript.counters == s2.transcript.counters
    assert s1.transcript.rounds == s2.transcript.rounds


@pytest.mark.parametrize("lanes", [7, 4096])
def test_batched_evaluator_against_plaintext(cuda, lanes):
    """Many input assignments per launch, including what the reference's
    evaluator cannot take: linear gates on online-only masks and MAXPOOL /
    DOT over wires with mixed P0 views (input next to truncation output)."""
    from paper_2411_09287_b200 import circuit
    text = ("INPUT 0 0\nINPUT 1 1\nINPUT 2 2\nCONST 3 384\n"
            "MUL 4 0 1\nTRUNC 5 4 8\nRELU 6 5\nADD 7 6 2\nSCALE 8 3 7\n"
            "MAXPOOL 9 3 0 5 8\nDOT 10 2 9 1 2 5\nTRUNC 11 10 8\nSUB 12 11 3\n"
            "OUTPUT 5\nOUTPUT 8\nOUTPUT 9\nOUTPUT 12")
    rng = np.random.default_rng(lanes)
    fx = lambda a: (np.trunc(a * 256).astype(np.int64)).astype(np.uint64)
    values = {w: fx(rng.normal(0, 3, lanes)) for w in (0, 1, 2)}
    _, res = _run(circuit.evaluate_batch, circuit.parse(text), values, lanes, 16, "auto", seed=lanes)
    outs, verdicts = res[0]
    assert all(verdicts.values())
    for o in res[1][0]:
        assert o.shape == (lanes,)
    want, bound = plain_eval_bounds(text, {w: [int(x) for x in v] for w, v in values.items()},
                                    lanes=lanes)
    for got, w, b in zip(outs, want, bound):
        d = np.abs(np.array([int(x) for x in got], dtype=object) - w)
        d = np.minimum(d, 2 ** 64 - d)
        assert np.all(d <= b)
    for role in (1, 2):
        for a, b in zip(res[role][0], outs):
            np.testing.assert_array_equal(a, b)


# ---------------------------------------------------------------------------
# CLI (tests/test_cli.py)
# ---------------------------------------------------------------------------

@pytest.fixture
def mul_circuit(tmp_path):
    p = tmp_path / "c.txt"
    p.write_text("INPUT 0 0\nINPUT 1 1\nMUL 2 0 1\nOUTPUT 2\n")
    return str(p)


def test_cli_simulate_and_transcript(cuda, mul_circuit, tmp_path, capsys):
    from paper_2411_09287_b200 import cli
    out = tmp_path / "t.csv"
    rc = cli.main(["simulate", mul_circuit, "--set", "0=6", "--set", "1=7", "--d", "16", "--R", "2",
                   "--seed", "5", "--transcript", str(out)])
    assert rc == cli.EXIT_OK
    assert "wire 2 = 42" in capsys.readouterr().out
    lines = out.read_text().splitlines()
    assert lines[0] == "from,to,phase,bytes,rounds" and len(lines) > 3


def test_cli_simulate_adversary_exit(cuda, mul_circuit):
    from paper_2411_09287_b200 import cli
    rc = cli.main(["simulate", mul_circuit, "--set", "0=6", "--set", "1=7", "--d", "16", "--R", "2",
                   "--seed", "5", "--adversary", "P0:gamma:+1"])
    assert rc == cli.EXIT_ABORT


def test_cli_config_error_exit(cuda):
    from paper_2411_09287_b200 import cli
    assert cli.main(["soundness", "--d", "3", "--trials", "1", "--gates", "2", "--seed", "1"]) == cli.EXIT_CONFIG


def test_cli_bench_formula_lines(cuda, capsys):
    from paper_2411_09287_b200 import cli
    assert cli.main(["bench", "mul", "--batch", "64", "--seed", "1"]) == cli.EXIT_OK
    out = capsys.readouterr().out
    assert "measured offline bits/op   64" in out and "measured online  bits/op   128" in out
    assert cli.main(["bench", "dot-trunc", "--n", "4", "--batch", "16", "--seed", "1"]) == cli.EXIT_OK
    assert "measured offline bits/op   448" in capsys.readouterr().out


def test_cli_soundness_csv_and_determinism(cuda, tmp_path, capsys):
    from paper_2411_09287_b200 import cli
    args = ["soundness", "--gates", "8", "--trials", "5", "--d", "16", "--R", "2", "--seed", "3",
            "--out", str(tmp_path / "s.csv")]
    assert cli.main(args) == cli.EXIT_OK
    first = (tmp_path / "s.csv").read_text()
    assert first.splitlines()[0] == "trial,injected_at,detected"
    assert cli.main(args) == cli.EXIT_OK
    assert (tmp_path / "s.csv").read_text() == first
    assert all(line.endswith(",1") for line in first.splitlines()[1:])
    err = capsys.readouterr().err
    assert "detection rate 1.0000 over 5 trials" in err
    # the reference's own report for these flags (its offline formula counts
    # fewer bits than its verification actually sends; reproduced as is)
    assert ("verification online bits: formula 15360 measured 15360; offline bits: "
            "formula 4096 measured 7168; rounds 4") in err


def test_cli_config_file_and_env_seed(cuda, tmp_path, mul_circuit, capsys, monkeypatch):
    from paper_2411_09287_b200 import cli
    cfgp = tmp_path / "cfg"
    cfgp.write_text("d=16\nR=1\nseed=9\n")
    assert cli.main(["--config", str(cfgp), "simulate", mul_circuit, "--set", "0=2", "--set", "1=3"]) == 0
    assert "wire 2 = 6" in capsys.readouterr().out
    monkeypatch.setenv("RING3PC_SEED", "77")
    assert cli.main(["simulate", mul_circuit, "--set", "0=2", "--set", "1=5", "--d", "16", "--R", "1"]) == 0
    assert "wire 2 = 10" in capsys.readouterr().out


def test_cli_infer(cuda, tmp_path, capsys):
    from paper_2411_09287_b200 import cli, ppml
    rng = np.random.default_rng(0)
    mp = tmp_path / "model.bin"
    ppml.save_model(str(mp), ppml.snn_model(rng))
    ip = tmp_path / "img.txt"
    ip.write_text("\n".join(str(v) for v in rng.normal(0, 1, 784)))
    rc = cli.main(["infer", "--model", str(mp), "--image", str(ip), "--d", "16", "--seed", "4", "--no-check"])
    assert rc == cli.EXIT_OK
    out = capsys.readouterr().out
    assert "argmax:" in out and "class 9:" in out


# ---------------------------------------------------------------------------
# statistical soundness (tests/test_acceptance.py:160-208), reduced trial count
# ---------------------------------------------------------------------------

def _trial_args(mode, t):
    rng = np.random.default_rng(40_000 + t)
    lane = int(rng.integers(0, 64))
    if mode == "random":
        return (1 << 20) + t, int(rng.integers(1, 1 << 63)), "z", lane
    if mode == "msb":
        return (2 << 20) + t, 1 << 63, "z", lane
    if mode == "gamma":
        return (3 << 20) + t, int(rng.integers(1, 1 << 63)), "gamma", lane
    return (4 << 20) + t, int(rng.integers(1, 1 << 63)), "mz", lane


def test_soundness_rates_reduced(cuda):
    """d = 16, R = 2, 64 gates: every injected error is detected (the
    criterion allows 3%); the d = 1 ring control accepts about half."""
    from paper_2411_09287_b200.cli import run_soundness_trial
    trials = 60
    for mode in ("random", "msb", "gamma", "mz"):
        miss = sum(not run_soundness_trial(*_trial_args(mode, t)[:1], 64, 16, 2, 64,
                                           *_trial_args(mode, t)[1:]) for t in range(trials))
        assert miss <= 2, (mode, miss)
    acc = sum(not run_soundness_trial((5 << 20) + t, 64, 1, 0, 64, 1 << 63, "gamma", 0)
              for t in range(200))
    assert 70 <= acc <= 130, acc
