"""The CLI mirrors the reference's subcommands, flags and exit codes (cli.py:1-250)."""
import pytest

from paper_1401_0248_b200.__main__ import build_parser, main


def test_parser_has_the_reference_subcommands():
    sub = build_parser()._subparsers._group_actions[0].choices
    assert set(sub) == {"accuracy", "hours100", "scaling", "bench", "read-baseline", "noread-baseline", "selftest"}


@pytest.mark.parametrize("argv", [["bench", "--methods", "bogus"], ["bench", "--flavor", "unroll:3"],
                                  ["read-baseline", "--channels", "3"], ["nope"], []])
def test_invalid_flags_exit_2(argv, capsys):
    assert main(argv) == 2


def test_flavor_parsing_accepts_cuda():
    args = build_parser().parse_args(["bench", "--flavor", "cuda", "--dot", "--tier", "small"])
    assert str(args.flavor) == "cuda" and args.dot and args.tier == ["small"]


@pytest.mark.gpu
@pytest.mark.parametrize("argv,needle", [
    (["selftest", "--no-meta"], "selftest: ok"),
    (["hours100", "--no-meta"], "twofold-fast"),
    (["accuracy", "--n", "100000", "--precision", "f32", "--generator", "nr", "--no-meta"], "twofold-fast"),
    (["scaling", "--n", "1000", "--n", "10000", "--trials", "3", "--no-meta"], "slope"),
    (["bench", "--tier", "small", "--precision", "f64", "--dot", "--repetitions", "3", "--no-meta"], "dottf"),
    (["read-baseline", "--tier", "small", "--channels", "2", "--no-meta"], "read2"),
    (["noread-baseline", "--methods", "twofold-fast", "--repetitions", "2", "--no-meta", "--format", "csv"],
     "psumtf"),
])
def test_subcommands_run_on_the_gpu(cuda, argv, needle, capsys):
    assert main(argv) == 0
    out = capsys.readouterr().out
    assert needle in out and not out.startswith("#")


@pytest.mark.gpu
def test_hours100_seq_reproduces_reference_goldens(cuda, golden, capsys):
    """accuracy.run_hours100 (test_acceptance.py:46-60) via the CLI: the seq flavor
    is bit-identical to the reference's own run (tests/golden/reference_outputs.json)."""
    assert main(["hours100", "--format", "csv", "--no-meta"]) == 0
    rows = {ln.split(",")[0]: ln.split(",")[1:] for ln in capsys.readouterr().out.strip().splitlines()[1:]}
    for g in golden["hours100"]:
        got = rows[g["method"]]
        assert float(got[0]) == float.fromhex(g["result_hours"]), g["method"]
        assert float(got[1]) == float.fromhex(g["deviation_hours"]), g["method"]
        if g["estimate_hours"] is not None:
            assert float(got[2]) == float.fromhex(g["estimate_hours"]), g["method"]


@pytest.mark.gpu
def test_no_meta_reruns_are_byte_identical(cuda, capsys):
    """cli.py:120-132 / test_cli.py:33-36: '#' metadata suppressed -> identical reports."""
    argv = ["accuracy", "--n", "50000", "--precision", "f64", "--format", "csv", "--no-meta"]
    assert main(argv) == 0
    first = capsys.readouterr().out
    assert main(argv) == 0
    assert capsys.readouterr().out == first and first.count("\n") == 1 + 2 * 2 * 3
