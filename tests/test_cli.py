"""CLI on the GPU path (reference cli.py:99-188): CSV interchange identical to
the reference, byte-deterministic runs, exit codes and error lines."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

import golden_cases as gc
from paper_2301_13441_b200.cli import format_f32, read_csv, run_cli, write_csv

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_csv_round_trip_and_formatting():
    x = np.array([[0, 1, -1.5], [1e-30, 3.4e38, 0.1], [np.nan, np.inf, -np.inf]], np.float32)
    text = write_csv(x)
    assert text.splitlines()[0] == "0.0,1.0,-1.5"  # the reference format_f32 (trim="0")
    back = read_csv(text, 3)
    assert np.array_equal(back, x, equal_nan=True)
    assert format_f32(np.float32(0.1)) == "0.1"
    assert read_csv("", 4).shape == (0, 4)


def test_bad_csv_is_a_validation_error(tmp_path, capsys):
    case = gc.get("sk_dt_d6")
    mp = tmp_path / "m.json"
    mp.write_text(case.entry["model_json"])
    inp = tmp_path / "x.csv"
    inp.write_text("1,2,x\n")
    assert run_cli(["run", "--model", str(mp), "--input", str(inp)]) == 2
    assert capsys.readouterr().err.startswith("error: validation:")


def test_unknown_pass_and_usage(tmp_path, capsys):
    assert run_cli(["run"]) == 2
    mp = tmp_path / "m.json"
    mp.write_text(gc.get("sk_dt_d6").entry["model_json"])
    assert run_cli(["compile", "--model", str(mp), "--passes", "re,zz"]) == 2


def test_missing_model_file(capsys):
    assert run_cli(["run", "--model", "/nonexistent.json", "--input", "/nonexistent.csv"]) == 2
    assert capsys.readouterr().err.startswith("error: io:")


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["sk_rf24_d8", "sk_logreg_784x10", "sk_gbr12_d6", "sk_standard_scaler"])
def test_run_matches_golden_and_is_byte_deterministic(name, tmp_path):
    case = gc.get(name)
    mp = tmp_path / "m.json"
    mp.write_text(case.entry["model_json"])
    inp = tmp_path / "x.csv"
    inp.write_text(write_csv(case.x))
    outs = []
    for k in range(2):
        op = tmp_path / f"y{k}.csv"
        r = subprocess.run([sys.executable, "-m", "paper_2301_13441_b200", "run", "--model", str(mp), "--input",
                            str(inp), "--output", str(op)], cwd=ROOT, capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        outs.append(op.read_bytes())
    assert outs[0] == outs[1]
    got = read_csv(outs[0].decode(), case.want.shape[1]).astype(np.float64)
    np.testing.assert_array_equal(got, case.want.astype(np.float32).astype(np.float64))


def test_json_profile_file(tmp_path, capsys):
    """--profile also takes a JSON profile (reference graph.py:146-168): a
    custom sparse_threshold reaches the lowering; a bad one is a ProfileError."""
    from paper_2301_13441_b200 import lower
    from paper_2301_13441_b200.errors import ProfileError
    good = tmp_path / "p.json"
    good.write_text('{"name": "dense", "preferred_int_dtype": "int16", "sparse_threshold": 0.0}')
    prof = lower.load_profile(str(good))
    assert prof.sparse_threshold == 0.0 and lower.sparse_threshold(str(good)) == 0.0
    bad = tmp_path / "bad.json"
    bad.write_text('{"name": "x", "preferred_int_dtype": "int16", "sparse_threshold": 1.5}')
    with pytest.raises(ProfileError):
        lower.load_profile(str(bad))
    with pytest.raises(ProfileError):
        lower.load_profile(str(tmp_path / "missing.json"))


REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "mlower")), reason="reference not installed in baseline/_ref")
@pytest.mark.parametrize("name", ["sk_rf24_d8", "sk_gbr12_d6", "sk_logreg_784x10"])
def test_verify_against_the_reference_oracle(name, tmp_path):
    """`verify` (reference cli.py:112-127) on the GPU path: boundary rows
    (one per threshold, cli.py:61-68) plus random rows, compared with the
    reference's own scalar oracle from the installed reference."""
    mp = tmp_path / "m.json"
    mp.write_text(gc.get(name).entry["model_json"])
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, ROOT]))
    r = subprocess.run([sys.executable, "-m", "paper_2301_13441_b200", "verify", "--model", str(mp), "--random", "300"],
                       cwd=ROOT, capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "result: PASS" in r.stdout
    assert "max_abs_divergence=0.0" in r.stdout or "mode=tolerance" in r.stdout
