"""CLI front end: flags, exit-code contract (cli.py:364-384) and, on a
GPU, `translate` end to end on a saved model directory vs the reference's
recorded records."""

import io
import json
import subprocess
import sys

import pytest

from conftest import GOLDEN, ROOT
from oracle.fixture_configs import CONFIGS, SEARCH_CASES


def test_help_and_no_command_exit_codes():
    proc = subprocess.run([sys.executable, "-m", "paper_2207_05851_b200", "--help"],
                          capture_output=True, text=True, cwd=ROOT)
    assert proc.returncode == 0 and "translate" in proc.stdout
    proc = subprocess.run([sys.executable, "-m", "paper_2207_05851_b200"],
                          capture_output=True, text=True, cwd=ROOT)
    assert proc.returncode == 1 and proc.stdout == ""


def test_out_of_scope_commands_exit_1(capsys):
    from paper_2207_05851_b200 import cli
    assert cli.main(["train"]) == 1
    assert cli.main(["translate", "-m", "/nonexistent/dir"]) == 2  # DataError


def _save_toy(tmp_path):
    from fixture_models import oracle_model, oracle_vocabs, product_config
    from paper_2207_05851_b200.checkpoint import Vocabulary, save_model_dir
    ov = oracle_vocabs("toy")
    v = Vocabulary(ov["trg"].tokens)
    save_model_dir(tmp_path / "toy", product_config("toy"), oracle_model("toy").p, v, v)
    return tmp_path / "toy"


@pytest.mark.gpu
def test_translate_cli_json_matches_reference(tmp_path, monkeypatch, capsys):
    from paper_2207_05851_b200 import cli
    mdir = _save_toy(tmp_path)
    case = next(c for c in SEARCH_CASES if c["name"] == "toy_beam3")
    gold = {c["name"]: c["records"] for c in
            json.loads((GOLDEN / "search.json").read_text())["cases"]}["toy_beam3"]
    lines = "\n".join(" ".join(i["tokens"]) for i in case["inputs"]) + "\n{bad json\n"
    monkeypatch.setattr(sys, "stdin", io.StringIO(lines))
    capsys.readouterr()
    assert cli.main(["translate", "-m", str(mdir), "--beam", "3", "--json",
                     "--precision", "fp32", "--batch-size", "4"]) == 0
    out = [json.loads(x) for x in capsys.readouterr().out.splitlines()]
    assert len(out) == len(gold) + 1
    assert "error" in out[-1] and out[-1]["translation"] == ""
    same = sum(o["translation"] == g["text"] for o, g in zip(out, gold))
    assert same == len(gold)


@pytest.mark.gpu
def test_bench_cli_reports_positive_rates(tmp_path, capsys):
    from paper_2207_05851_b200 import cli
    mdir = _save_toy(tmp_path)
    capsys.readouterr()
    assert cli.main(["bench", "-m", str(mdir), "--sentences", "2", "--steps", "6",
                     "--warmup", "1", "--length", "5"]) == 0
    vals = dict(line.split(" = ") for line in capsys.readouterr().out.splitlines())
    assert set(vals) == {"sentences_per_sec", "tokens_per_sec", "decoder_step_cost"}
    assert all(float(v) > 0 for v in vals.values())


@pytest.mark.gpu
def test_translate_cli_quantized_int8(tmp_path, monkeypatch, capsys):
    """`translate --quantize int8` (cli.py:130-131): the feed-forward layers
    run on the int8 path and every line still gets a translation."""
    from paper_2207_05851_b200 import cli
    mdir = _save_toy(tmp_path)
    monkeypatch.setattr(sys, "stdin", io.StringIO("w1 w2 w3\nw4 w5\n"))
    capsys.readouterr()
    assert cli.main(["translate", "-m", str(mdir), "--quantize", "int8", "--json"]) == 0
    out = [json.loads(x) for x in capsys.readouterr().out.splitlines()]
    assert len(out) == 2 and all("error" not in o for o in out)
