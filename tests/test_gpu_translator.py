"""Translator facade on the GPU vs the reference's text pipeline composed
around the reference model (tests/golden/translator.json, made by
oracle/make_golden_text.py), plus the reference's engine/CLI contracts
(tests/test_engine_cli.py:26-233 of the reference)."""

import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import nmt_oracle as O  # noqa: E402
from oracle import parity as P  # noqa: E402
from paper_2109_08003_b200 import modelfile as MF  # noqa: E402
from paper_2109_08003_b200 import store as S  # noqa: E402
from paper_2109_08003_b200 import textpipe as T  # noqa: E402
from paper_2109_08003_b200.translator import RunConfig, Translator  # noqa: E402

G = Path(__file__).resolve().parent / "golden"
ROOT = G.parent.parent
TR = json.loads((G / "translator.json").read_text())
TX = json.loads((G / "textpipe.json").read_text())


def assets():
    codec = T.BpeCodec([tuple(m) for m in TX["merges"]])
    vocab = T.Vocabulary(TX["vocab"][4:])
    c = TR["cfg"]
    cfg = S.ModelConfig(n_enc_layers=2, n_dec_layers=1, d_model=c["d_model"], n_heads_enc=2,
                        n_heads_dec=1, ffn_dim_enc=32, ffn_dim_dec=16,
                        vocab_size=c["vocab_size"], max_positions=c["max_positions"])
    return cfg, S.random_model(cfg, TR["seed"]), vocab, codec


@pytest.fixture(scope="module")
def tr32():
    cfg, w, vocab, codec = assets()
    return Translator(cfg, w, vocab, codec=codec, run=RunConfig(precision="f32"))


@pytest.fixture(scope="module")
def tr16():
    cfg, w, vocab, codec = assets()
    return Translator(cfg, w, vocab, codec=codec, run=RunConfig(precision="f16"))


def test_f32_lines_identical_to_reference(tr32):
    assert tr32.translate_lines(TR["lines"]) == TR["greedy"]


def test_f32_beam_pretok_nocodec_identical(tr32):
    assert tr32.with_run(beam=2).translate_lines(TR["lines"][:12]) == TR["beam2"]
    assert tr32.with_run(pretokenized=True).translate_lines(TR["lines"][:12]) == TR["pretok"]
    nc = Translator(tr32.cfg, tr32.weights, tr32.vocab, codec=None, run=RunConfig(precision="f32"))
    assert nc.translate_lines(TR["lines"][:12]) == TR["nocodec"]


def test_f16_lines_identical_or_near_tie(tr16):
    """fp16 text lines: every line whose subword ids match the oracle's greedy
    ids is identical to the reference's line, and every id divergence is a
    near-tie of the oracle's logits (oracle/parity.py)."""
    got = tr16.translate_lines(TR["lines"])
    assert len(got) == len(TR["lines"])
    chunk = tr16._to_ids(TR["lines"])
    got_ids = [x.tolist() for x in tr16._translate_pieces(chunk.pieces)]
    a = O.arch_of(tr16.cfg)
    p = O.make_params(a, TR["seed"])
    want_ids = []
    for i in range(0, len(chunk.pieces), 16):
        rows = [r.astype(np.int64) for r in chunk.pieces[i:i + 16]]
        live = [j for j, r in enumerate(rows) if len(r)]
        outs = O.greedy(a, p, *O.pad_rows([rows[j] for j in live])) if live else []
        res = [[] for _ in rows]
        for j, o in zip(live, outs):
            res[j] = o
        want_ids += res
    rep = P.near_tie_report(a, p, [r.astype(np.int64) for r in chunk.pieces], got_ids, want_ids)
    print("translator fp16 ids:", rep)
    assert rep["all_near_ties"], rep
    same_ids = {li for li, g, w in zip(chunk.owner, got_ids, want_ids) if g == w}
    bad_ids = {li for li, g, w in zip(chunk.owner, got_ids, want_ids) if g != w}
    for li in same_ids - bad_ids:
        assert got[li] == TR["greedy"][li], li


def test_line_contract(tr16):
    lines = ["the quick fox", "", "lazy dog.", "", ""]
    out = tr16.translate_lines(lines)
    assert len(out) == 5 and out[1] == out[3] == out[4] == ""
    assert tr16.translate_lines([]) == []
    out = tr16.translate_lines(["the quick brown fox " * 600, "short one"])
    assert len(out) == 2 and out[0] != ""


@pytest.mark.parametrize("workers", [2, 4, 8])
def test_worker_and_cap_invariance(tr16, workers):
    rng = np.random.default_rng(1)
    words = ["the", "quick", "brown", "fox", "lazy", "dog", "river", "stone"]
    lines = [" ".join(rng.choice(words, size=int(rng.integers(1, 9)))) for _ in range(40)]
    seq = tr16.with_run(workers=1, chunk_lines=7).translate_lines(lines)
    assert tr16.with_run(workers=workers, chunk_lines=7).translate_lines(lines) == seq
    assert tr16.with_run(sbatch=1, wbatch=16).translate_lines(lines) == seq
    assert tr16.with_run(sbatch=8, wbatch=128, chunk_lines=5).translate_lines(lines) == seq


def test_bench_report(tr16):
    rng = np.random.default_rng(6)
    lines = [" ".join(["the", "fox"] * int(rng.integers(1, 5))) for _ in range(25)]
    rep = tr16.bench(lines)
    words = sum(len(x.split()) for x in lines)
    assert rep["source_words"] == words and rep["source_sentences"] == 25
    assert rep["output_lines"] == 25
    assert rep["words_per_second"] == pytest.approx(words / rep["wall_seconds"], rel=1e-9)
    assert rep["est_peak_bytes"] > 0
    for k in ("sbatch", "wbatch", "workers", "chunk_lines", "precision"):
        assert k in rep


def test_selftest_battery(tr16):
    res = tr16.selftest()
    assert all(ok for _, ok, _ in res), res
    names = [n for n, _, _ in res]
    assert "very_long_line" in names and "dirty_bytes" in names


def test_from_reference_model_file():
    t = Translator.from_file(G / "model_f32.fnmt", run=RunConfig(precision="f32"))
    out = t.translate_lines(["w4 w5", "", "!"])
    assert len(out) == 3 and out[1] == ""


def run_cli(*args, stdin=b""):
    return subprocess.run([sys.executable, "-m", "paper_2109_08003_b200.cli", *args], input=stdin,
                          capture_output=True, timeout=300, cwd=ROOT)


def test_cli_translate_bench_selftest(tmp_path):
    m = G / "model_f32.fnmt"
    r = run_cli("translate", "--model", str(m), stdin=b"hello world\n\nsecond line\n")
    assert r.returncode == 0, r.stderr
    assert r.stdout.decode().split("\n")[1] == "" and len(r.stdout.decode().splitlines()) == 3
    r = run_cli("translate", "--model", str(m), stdin=b"")
    assert r.returncode == 0 and r.stdout == b""
    corpus = tmp_path / "c.txt"
    corpus.write_text("one two three\nfour five\n" * 10)
    r = run_cli("bench", "--model", str(m), "--corpus", str(corpus), "--precision", "f32")
    assert r.returncode == 0, r.stderr
    rep = dict(x.split("=", 1) for x in r.stdout.decode().splitlines() if "=" in x)
    assert int(rep["source_words"]) == 50 and rep["precision"] == "f32"
    assert float(rep["words_per_second"]) > 0
    r = run_cli("selftest")
    assert r.returncode == 0, r.stdout + r.stderr
    assert b"selftest=pass" in r.stdout


def test_multi_engine_translate_identical(tr16):
    """devices=(0, 0): two engines (the multi-GPU layout, here on one GPU) with
    chunk groups round-robin — output identical to one engine."""
    cfg, w, vocab, codec = assets()
    lines = TR["lines"] * 3
    one = tr16.with_run(chunk_lines=5).translate_lines(lines)
    import paper_2109_08003_b200.translator as trm
    old = trm.GPU_GROUP_LINES
    trm.GPU_GROUP_LINES = 10          # several groups per engine
    try:
        two = Translator(cfg, w, vocab, codec=codec,
                         run=RunConfig(precision="f16", chunk_lines=5, devices=(0, 0)))
        assert two.translate_lines(lines) == one
        assert two.bench(lines[:10])["devices"] == 2
    finally:
        trm.GPU_GROUP_LINES = old
