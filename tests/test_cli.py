"""Device CLI vs the reference CLI (cli.py): exit codes, formats, identical outputs."""

import json

import pytest

from _cli_cases import run_cli
from _specs import load_json
from paper_2604_17066_b200.cli import TRACE_COLUMNS, main


def test_missing_subcommand_is_usage_error():
    with pytest.raises(SystemExit) as exc:
        main([])
    assert exc.value.code == 2


def test_unknown_flag_is_usage_error(tmp_path):
    with pytest.raises(SystemExit) as exc:
        main(["oracle", "--model", str(tmp_path / "m.json"), "--mode", "exact", "--bogus"])
    assert exc.value.code == 2


def test_missing_and_malformed_model_are_input_errors(tmp_path, capsys):
    code = main(["find-refs", "--model", str(tmp_path / "nope.json"), "--out-refs",
                 str(tmp_path / "r.json")])
    assert code == 3 and "error:" in capsys.readouterr().err
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    assert main(["oracle", "--model", str(bad), "--mode", "exact"]) == 3


def test_gen_graph_matches_reference(tmp_path, reference_rsr):
    from rsr.cli import main as ref_main
    a, b = tmp_path / "a.json", tmp_path / "b.json"
    assert main(["gen-graph", "--n-nodes", "12", "--radius", "0.5", "--out", str(a), "--seed", "3"]) == 0
    assert ref_main(["gen-graph", "--n-nodes", "12", "--radius", "0.5", "--out", str(b),
                     "--seed", "3"]) == 0
    da, db = json.loads(a.read_text()), json.loads(b.read_text())
    for d in (da, db):
        d["manifest"].pop("timestamp")
        d["manifest"].pop("tool_version")
    assert da == db


def test_trace_columns_match_reference(reference_rsr):
    from rsr.cli import TRACE_COLUMNS as REF
    assert TRACE_COLUMNS == REF


@pytest.mark.gpu
def test_cli_runs_match_reference_outputs(tmp_path):
    # tests/golden/cli.json: the same command lines run through the reference CLI
    got = run_cli(main, str(tmp_path))
    want = load_json("cli.json")
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert g["code"] == w["code"] == 0
        assert g.get("trace") == w.get("trace")
        assert g["out"] == w["out"]
