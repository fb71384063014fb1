"""Host-only CLI subcommands (no GPU needed): inspect, random-model, load
errors (reference tests/test_engine_cli.py:171-233)."""

import subprocess
import sys
from pathlib import Path

from paper_2109_08003_b200 import modelfile as MF
from paper_2109_08003_b200.translator import RunConfig

import pytest

ROOT = Path(__file__).resolve().parent.parent
G = ROOT / "tests" / "golden"


def run_cli(*args, stdin=b""):
    return subprocess.run([sys.executable, "-m", "paper_2109_08003_b200.cli", *args], input=stdin,
                          capture_output=True, timeout=300, cwd=ROOT)


def test_inspect():
    r = run_cli("inspect", "--model", str(G / "model_f32.fnmt"))
    assert r.returncode == 0
    assert b"src_embed" in r.stdout and b"config:" in r.stdout


def test_missing_model_exits_2(tmp_path):
    r = run_cli("translate", "--model", str(tmp_path / "missing.fnmt"), stdin=b"x\n")
    assert r.returncode == 2
    assert b"cannot load model" in r.stderr


@pytest.mark.parametrize("prec", ["f32", "int8"])
def test_random_model_generation(tmp_path, prec):
    out = tmp_path / "gen.fnmt"
    r = run_cli("random-model", "--out", str(out), "--d-model", "32", "--enc-layers", "2",
                "--ffn-enc", "64", "--ffn-dec", "32", "--vocab-size", "64", "--max-positions",
                "64", "--heads-enc", "2", "--precision", prec)
    assert r.returncode == 0, r.stderr
    cfg, w, vocab = MF.load(out, precision=prec)
    assert cfg.d_model == 32 and len(vocab) == 64


def test_run_config_validation():
    with pytest.raises(ValueError):
        RunConfig(precision="f64")
    with pytest.raises(ValueError):
        RunConfig(workers=0)
    assert RunConfig().sbatch == 3072 and RunConfig().wbatch == 64000
