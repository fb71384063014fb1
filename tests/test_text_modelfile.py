"""Host pipeline parity (CPU): text pipeline and FNMT model files against
fixtures produced by the reference itself (oracle/make_golden_text.py)."""

import json
from pathlib import Path

import numpy as np
import pytest

from paper_2109_08003_b200 import modelfile as MF
from paper_2109_08003_b200 import quant8 as Q
from paper_2109_08003_b200 import store as S
from paper_2109_08003_b200 import textpipe as T

G = Path(__file__).resolve().parent / "golden"
TEXT = json.loads((G / "textpipe.json").read_text())


def codec():
    return T.BpeCodec([tuple(m) for m in TEXT["merges"]])


def test_tokenize_matches_reference():
    for line, want in zip(TEXT["lines"], TEXT["tokenize"]):
        assert T.tokenize(line) == want, line


def test_detokenize_matches_reference():
    for line, want in zip(TEXT["lines"], TEXT["detokenize"]):
        assert T.detokenize(T.tokenize(line)) == want, line


def test_tokenize_idempotent_and_total():
    rng = np.random.default_rng(0)
    for _ in range(200):
        raw = bytes(rng.integers(0, 256, size=int(rng.integers(0, 60)), dtype=np.uint8))
        line = raw.decode("utf-8", errors="replace")
        toks = T.tokenize(line)
        assert T.tokenize(" ".join(toks)) == toks


def test_bpe_segment_and_encode_match_reference():
    c = codec()
    for w, want in zip(TEXT["segment_words"], TEXT["segment"]):
        assert c.segment(w) == want, w
        assert c.segment(w) == want            # memoised path
    for line, want in zip(TEXT["lines"], TEXT["bpe_encode"]):
        assert T.bpe_encode(T.tokenize(line), c) == want


def test_bpe_decode_matches_reference():
    for pieces, want in zip(TEXT["bpe_decode_in"], TEXT["bpe_decode"]):
        assert T.bpe_decode(pieces) == want


def test_bpe_roundtrip():
    c = codec()
    for line in TEXT["lines"]:
        toks = T.tokenize(line)
        assert T.bpe_decode(T.bpe_encode(toks, c)) == toks


def test_vocab_and_synthetic_vocab(tmp_path):
    v = T.Vocabulary(TEXT["vocab"][4:])
    assert v.all_tokens() == TEXT["vocab"]
    assert T.synthetic_vocabulary(10).all_tokens() == TEXT["synthetic_vocab_10"]
    assert T.synthetic_vocabulary(100).all_tokens() == TEXT["synthetic_vocab_100"]
    assert v.id_of("never-seen") == T.UNK_ID and v.token_of(10 ** 6) == "<unk>"
    v.save(tmp_path / "v.txt")
    assert T.Vocabulary.load(tmp_path / "v.txt").all_tokens() == v.all_tokens()
    (tmp_path / "bad.txt").write_text("a 4\nb 6\n")
    with pytest.raises(ValueError):
        T.Vocabulary.load(tmp_path / "bad.txt")


def test_codes_file_roundtrip(tmp_path):
    c = codec()
    c.save(tmp_path / "codes")
    assert T.BpeCodec.load(tmp_path / "codes") == c
    (tmp_path / "w").write_text("#version: 0.2\na b</w>\nx\n\nc d\n")
    assert T.BpeCodec.load(tmp_path / "w").merges == [("a", "b"), ("c", "d")]


def test_run_parallel_order_and_failure():
    lines = [str(i) for i in range(50)]
    for workers in (1, 3, 8):
        plan = T.ChunkPlan.for_lines(len(lines), 7, workers)
        assert T.run_parallel(lines, plan, lambda ch: [x + "!" for x in ch]) == [
            x + "!" for x in lines]

    def bad(ch):
        if "22" in ch:
            raise RuntimeError("boom")
        return ch
    with pytest.raises(T.ChunkFailure) as e:
        T.run_parallel(lines, T.ChunkPlan.for_lines(50, 7, 4), bad)
    assert e.value.chunk_index == 3
    with pytest.raises(T.ChunkFailure):
        T.run_parallel(lines, T.ChunkPlan.for_lines(50, 7, 1), lambda ch: ch[:-1])
    with pytest.raises(ValueError):
        T.ChunkPlan.for_lines(5, 0, 1)


# ---------------------------------------------------------------------------
# model files

def ref_like_model(seed, **kw):
    cfg = S.ModelConfig(**{**dict(n_enc_layers=2, n_dec_layers=1, d_model=16, n_heads_enc=2,
                                  n_heads_dec=1, ffn_dim_enc=32, ffn_dim_dec=16, vocab_size=100,
                                  max_positions=64), **kw})
    return cfg, S.random_model(cfg, seed)


@pytest.mark.parametrize("name,prec,seed,kw", [
    ("model_f32.fnmt", "f32", 9, {}),
    ("model_int8.fnmt", "int8", 9, {}),
    ("model_unshared_int8.fnmt", "int8", 10,
     dict(shared_embeddings=False, n_dec_layers=2, ffn_dim_dec=0)),
    ("model_unshared_f32.fnmt", "f32", 10,
     dict(shared_embeddings=False, n_dec_layers=2, ffn_dim_dec=0)),
])
def test_save_is_byte_identical_to_reference(tmp_path, name, prec, seed, kw):
    cfg, w = ref_like_model(seed, **kw)
    out = tmp_path / name
    MF.save(w, cfg, out, precision=prec, vocab=T.synthetic_vocabulary(100))
    assert out.read_bytes() == (G / name).read_bytes()


def test_load_reference_files():
    cfg, w = ref_like_model(9)
    c2, w2, v2 = MF.load(G / "model_f32.fnmt")
    assert c2 == cfg and v2.all_tokens() == T.synthetic_vocabulary(100).all_tokens()
    for (n1, a1), (n2, a2) in zip(S.iter_named_tensors(cfg, w), S.iter_named_tensors(c2, w2)):
        assert n1 == n2 and np.array_equal(a1, a2), n1
    # int8 file at int8 precision: quantized weights equal quantize-at-load of the f32 file
    _, wq, _ = MF.load(G / "model_int8.fnmt", precision="int8")
    _, wq2, _ = MF.load(G / "model_f32.fnmt", precision="int8")
    a, b = wq.enc_layers[0].attn.q.weight, wq2.enc_layers[0].attn.q.weight
    assert isinstance(a, Q.QuantizedMatrix)
    assert np.array_equal(a.q, b.q) and np.array_equal(a.col_scale, b.col_scale)
    assert np.array_equal(wq.out_proj.weight.q, wq2.out_proj.weight.q)
    # int8 file at f32 precision: dequantized (lossy) weights
    _, wd, _ = MF.load(G / "model_int8.fnmt", precision="f32")
    ref = w.enc_layers[0].attn.q.weight
    got = wd.enc_layers[0].attn.q.weight
    assert got.dtype == np.float32 and np.abs(got - ref).max() < 0.05


def test_describe_matches_reference():
    d = MF.describe(G / "model_f32.fnmt").splitlines()[1:]
    assert d == TEXT["models"]["describe_f32"]


def test_load_rejects_corrupt_files(tmp_path):
    raw = (G / "model_f32.fnmt").read_bytes()
    bad = tmp_path / "bad.fnmt"
    bad.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(MF.ModelFormatError, match="bad magic"):
        MF.load(bad)
    bad.write_bytes(raw[:4] + (2).to_bytes(4, "little") + raw[8:])
    with pytest.raises(MF.ModelFormatError, match="unsupported version"):
        MF.load(bad)
    bad.write_bytes(raw[:-10])
    with pytest.raises(MF.ModelFormatError, match="truncated"):
        MF.load(bad)
    with pytest.raises(OSError):
        MF.load(tmp_path / "missing.fnmt")
    with pytest.raises(ValueError):
        MF.load(G / "model_f32.fnmt", precision="f64")


def test_quantize_weights_properties():
    rng = np.random.default_rng(1)
    w = (rng.standard_normal((64, 40)) * 0.1 + 0.02).astype(np.float32)
    w[:, 3] = 0.25                                    # degenerate column
    qm = Q.quantize_weights(w)
    dq = Q.dequantize_weights(qm)
    assert np.array_equal(dq[:, 3], w[:, 3])
    inside = np.abs(w - w.mean(0)) < 7 * w.std(0)
    err = np.abs(dq - w)
    assert np.all(err[inside] <= (qm.col_scale[None, :] / 2 + 1e-6).repeat(64, 0)[inside])
