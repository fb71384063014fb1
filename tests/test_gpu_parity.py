"""End-to-end parity of the CUDA engine against the reference / oracle.

Tolerances (BASELINE.json north_star):
  * fp32 parity mode: encoder states and logits within 1e-4 relative
    (|got - want| <= 1e-4 * max(1, max|want|)), greedy ids identical;
  * fp16: logits within 1e-2 (same relative form), greedy outputs
    token-identical on >= 99% of sentences, every divergence a near-tie
    (reference top-1/top-2 logit gap <= 0.05 at the first divergent step).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import nmt_oracle as O  # noqa: E402
from oracle import parity as P  # noqa: E402
from paper_2109_08003_b200 import store as S  # noqa: E402
from paper_2109_08003_b200.engine import Engine  # noqa: E402
from paper_2109_08003_b200.model import GpuTranslationModel  # noqa: E402
from paper_2109_08003_b200.search import SearchConfig, beam_translate, greedy_translate  # noqa: E402

CASES = ["tiny", "tiny_dec2_h2", "tiny_noffn", "tiny_l1", "tiny_unshared", "d32_student",
         "d64_h8_dec6", "d64_h1_l1"]
SC = SearchConfig(bos_id=2, eos_id=3, pad_id=0)


def rel_err(got, want):
    return float(np.abs(np.asarray(got) - np.asarray(want)).max() / max(1.0, np.abs(want).max()))


def split(ids, lens):
    out, o = [], 0
    for n in lens:
        out.append([int(x) for x in ids[o:o + n]])
        o += int(n)
    return out


def case(golden, tag):
    g = golden("small_models")
    get = lambda k: g[f"{tag}__{k}"]
    c = [int(x) for x in get("config")]
    cfg = S.ModelConfig(*c[:9], norm_variant="l1" if c[9] else "l2", shared_embeddings=bool(c[10]))
    return cfg, S.random_model(cfg, int(get("seed"))), get


@pytest.mark.parametrize("tag", CASES)
def test_fp32_protocol_matches_reference(golden, tag):
    cfg, w, get = case(golden, tag)
    m = GpuTranslationModel(cfg, w, dtype="f32")
    tok, valid = get("tokens"), get("valid")
    enc = m.encode(tok, valid)
    assert rel_err(enc.states, get("states")) <= 1e-4
    cache = m.init_cache(enc)
    prev = np.full(tok.shape[0], 2, np.int64)
    for t in range(6):
        logits = m.step(cache, prev)
        assert rel_err(logits, get("logits")[t]) <= 1e-4, t
        prev = get("forced")[:, t]
    assert greedy_translate(m, enc, SC) == split(get("greedy_ids"), get("greedy_lens"))
    for k in (1, 2, 4):
        cfgk = SearchConfig(2, 3, 0, beam_size=k)
        assert beam_translate(m, enc, cfgk) == split(get(f"beam{k}_ids"), get(f"beam{k}_lens"))


@pytest.mark.parametrize("tag", CASES)
def test_fp16_logits_within_tolerance(golden, tag):
    cfg, w, get = case(golden, tag)
    m = GpuTranslationModel(cfg, w, dtype="f16")
    tok, valid = get("tokens"), get("valid")
    enc = m.encode(tok, valid)
    cache = m.init_cache(enc)
    prev = np.full(tok.shape[0], 2, np.int64)
    for t in range(6):
        assert rel_err(m.step(cache, prev), get("logits")[t]) <= 1e-2, t
        prev = get("forced")[:, t]


def test_protocol_loop_equals_fused_decode(golden):
    """The reference's greedy algorithm driven through step() (protocol path)
    gives the same ids as the fused device decode (graph + argmax epilogue)."""
    cfg, w, get = case(golden, "d64_h8_dec6")
    for dtype in ("f32", "f16"):
        m = GpuTranslationModel(cfg, w, dtype=dtype)
        enc = m.encode(get("tokens"), get("valid"))
        fused = greedy_translate(m, enc, SC)
        lens = get("valid").sum(axis=1)
        budgets = [max(1, min(cfg.max_positions, int(np.ceil(1.5 * n)) + 5)) for n in lens]
        cache = m.init_cache(enc)
        feed = np.full(len(lens), 2, np.int64)
        done = np.zeros(len(lens), bool)
        outs = [[] for _ in lens]
        for t in range(max(budgets)):
            m.step(cache, feed)
            best = m.last_step_argmax()
            feed = np.zeros(len(lens), np.int64)
            for r in range(len(lens)):
                if done[r]:
                    continue
                if best[r] == 3:
                    done[r] = True
                    continue
                outs[r].append(int(best[r]))
                feed[r] = best[r]
                done[r] = t + 1 >= budgets[r]
            if done.all():
                break
        assert outs == fused, dtype


def test_engine_batch_caps_do_not_change_output(golden):
    """Byte-identical outputs across batch plans (reference acceptance
    'batching-invariance', tests/test_acceptance.py:220-242)."""
    cfg, w, get = case(golden, "d32_student")
    eng = Engine(cfg, w, dtype="f16")
    rng = np.random.default_rng(7)
    rows = [rng.integers(4, cfg.vocab_size, size=int(rng.integers(1, 30))) for _ in range(300)]
    lengths = np.array([len(r) for r in rows])
    offsets = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    ids = np.concatenate(rows).astype(np.int32)
    results = []
    for sb, wb in [(1, 16), (8, 128), (128, 2048), (3072, 64000)]:
        out, olen, off, st = eng.translate(ids, offsets, sbatch=sb, wbatch=wb)
        results.append(split_off(out, olen, off))
    assert results[0] == results[1] == results[2] == results[3]
    # oracle greedy on a slice (f16 near-ties aside, tiny vocab: compare f32 engine)
    eng32 = Engine(cfg, w, dtype="f32")
    out, olen, off, _ = eng32.translate(ids[:offsets[20]], offsets[:21])
    a = O.arch_of(cfg)
    p = O.make_params(a, int(get("seed")))
    tok, valid = O.pad_rows(rows[:20])
    assert split_off(out, olen, off) == O.greedy(a, p, tok, valid)


def split_off(out, olen, off):
    return [out[o:o + n].tolist() for o, n in zip(off, olen)]


@pytest.fixture(scope="module")
def student_weights():
    cfg = S.ModelConfig(6, 1, 512, 1, 1, 2048, 2048, 32772, 1024)
    return cfg, S.random_model(cfg, 0)


@pytest.mark.parametrize("dtype", ["f32", "f16"])
def test_config1_student_greedy_vs_reference(golden, student_weights, dtype):
    """BASELINE config 1: Student-6-1-1, 64 synthetic sentences, reference ids."""
    g = golden("config1_greedy")
    cfg, w = student_weights
    rows = O.config1_sentences()
    want = split(g["out_ids"], g["out_lens"])
    lengths = np.array([len(r) for r in rows])
    offsets = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    eng = Engine(cfg, w, dtype=dtype)
    out, olen, off, st = eng.translate(np.concatenate(rows).astype(np.int32), offsets,
                                       sbatch=128, wbatch=2048)
    got = split_off(out, olen, off)
    same = sum(a == b for a, b in zip(got, want))
    if dtype == "f32":
        assert same == 64
        return
    # near-tie report for every divergence
    starts = np.concatenate([[0], np.cumsum(g["step_counts"])])
    report = []
    for i, (a, b) in enumerate(zip(got, want)):
        if a == b:
            continue
        j = next(j for j in range(min(len(a), len(b))) if a[j] != b[j])
        gap = float(g["top1"][starts[i] + j] - g["top2"][starts[i] + j])
        report.append((i, j, gap))
    print("fp16 divergences (sentence, step, reference top1-top2 gap):", report)
    # 64 sentences: every divergence must be a near-tie (the >= 99% identical
    # rate is asserted at corpus scale, test_gpu_corpus_parity.py)
    assert all(gap <= P.NEAR_TIE for _, _, gap in report), report


@pytest.mark.parametrize("d,heads,dec", [(256, 4, 1), (512, 4, 2), (512, 2, 1), (512, 8, 1),
                                         (256, 2, 1), (768, 8, 2), (256, 8, 1), (1024, 8, 1)])
def test_multihead_decode_rows_fp16(d, heads, dec):
    """Decoder shapes that take the all-heads-per-row decode attention
    (head sizes 64 / 128 / 256 in fp16): logits of 6 forced steps within the
    fp16 tolerance of the oracle, and native beam-4 (ancestor-table self
    attention) close to the oracle's beam.  (768, 8) and (256, 8) have head
    sizes 96 / 32 whose lane groups are not powers of two (smem partials)."""
    cfg = S.ModelConfig(2, dec, d, heads, heads, 2 * d, d, 300, 64)
    seed = d + heads + dec
    w = S.random_model(cfg, seed)
    a = O.arch_of(cfg)
    p = O.make_params(a, seed)
    rng = np.random.default_rng(seed)
    rows = [rng.integers(4, cfg.vocab_size, size=int(rng.integers(3, 20))) for _ in range(9)]
    tok, valid = O.pad_rows(rows)
    m = GpuTranslationModel(cfg, w, dtype="f16")
    enc = m.encode(tok, valid)
    cache = m.init_cache(enc)
    oc = O.start_cache(a, p, O.encoder(a, p, tok, valid), valid)
    prev = np.full(len(rows), 2, np.int64)
    for t in range(6):
        want = O.decoder_step(a, p, oc, prev)
        assert rel_err(m.step(cache, prev), want) <= 1e-2, t
        prev = want.argmax(axis=1).astype(np.int64)
    eng = Engine(cfg, w, dtype="f16")
    lengths = np.array([len(r) for r in rows])
    offsets = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    out, olen, off, _ = eng.translate(np.concatenate(rows).astype(np.int32), offsets, beam=4)
    got = split_off(out, olen, off)
    want = O.beam(a, p, tok, valid, 4)
    rep = P.near_tie_report(a, p, rows, got, want, beam=4)
    assert rep["all_near_ties"], rep


@pytest.mark.parametrize("tag", ["tiny", "d32_student", "d64_h8_dec6", "d64_h1_l1"])
def test_bf16_logits_within_tolerance(golden, tag):
    """bf16 storage (the Deep-12-768 configuration's dtype): logits of forced
    decode steps within 2e-2 relative of the reference (bf16 keeps 8 mantissa
    bits vs fp16's 11, so the fp16 bound of 1e-2 is doubled)."""
    cfg, w, get = case(golden, tag)
    m = GpuTranslationModel(cfg, w, dtype="bf16")
    tok, valid = get("tokens"), get("valid")
    enc = m.encode(tok, valid)
    assert rel_err(enc.states, get("states")) <= 2e-2
    cache = m.init_cache(enc)
    prev = np.full(tok.shape[0], 2, np.int64)
    for t in range(6):
        assert rel_err(m.step(cache, prev), get("logits")[t]) <= 2e-2, t
        prev = get("forced")[:, t]


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
def test_folded_cross_attention_corpus_path(dtype):
    """Single-head decoders with d % 256 == 0 run the folded cross attention in
    the corpus path (K Wq^T / V Wo / bq.k precomputed per batch, no per-step
    cross-q / cross-o GEMMs): greedy and beam-4 outputs agree with the oracle
    (the protocol path, which keeps the unfolded GEMMs, is checked on logits
    elsewhere)."""
    cfg = S.ModelConfig(2, 1, 256, 2, 1, 512, 256, 400, 64)
    w = S.random_model(cfg, 11)
    a = O.arch_of(cfg)
    p = O.make_params(a, 11)
    rng = np.random.default_rng(11)
    rows = [rng.integers(4, cfg.vocab_size, size=int(rng.integers(2, 25))) for _ in range(40)]
    tok, valid = O.pad_rows(rows)
    lengths = np.array([len(r) for r in rows])
    offsets = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    ids = np.concatenate(rows).astype(np.int32)
    eng = Engine(cfg, w, dtype=dtype)
    tie = P.NEAR_TIE if dtype == "f16" else P.NEAR_TIE_BF16
    for k, want in ((1, O.greedy(a, p, tok, valid)), (4, O.beam(a, p, tok, valid, 4))):
        out, olen, off, _ = eng.translate(ids, offsets, beam=k)
        got = split_off(out, olen, off)
        # 40 sentences: every divergence must be a near-tie (the >= 99% rate is
        # asserted at corpus scale, test_gpu_corpus_parity.py)
        rep = P.near_tie_report(a, p, rows, got, want, beam=k, near_tie=tie)
        print(dtype, k, rep)
        assert rep["all_near_ties"], (k, rep)


def test_engine_translate_absolute_offsets(golden):
    """fnmt_engine_translate reads sentence i at ids[offsets[i]:offsets[i+1]]
    with absolute offsets into the caller's array (include/fnmt_b200.h): a
    slice of a corpus passed with its absolute offsets equals the rebased call."""
    cfg, w, get = case(golden, "d32_student")
    eng = Engine(cfg, w, dtype="f16")
    rng = np.random.default_rng(3)
    rows = [rng.integers(4, cfg.vocab_size, size=int(rng.integers(1, 20))) for _ in range(60)]
    lengths = np.array([len(r) for r in rows])
    offsets = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    ids = np.concatenate(rows).astype(np.int32)
    lo, hi = 25, 60
    a, alen, aoff, _ = eng.translate(ids, offsets[lo:hi + 1])
    b, blen, boff, _ = eng.translate(ids[offsets[lo]:offsets[hi]].copy(),
                                     offsets[lo:hi + 1] - offsets[lo])
    assert split_off(a, alen, aoff) == split_off(b, blen, boff)
    full, flen, foff, _ = eng.translate(ids, offsets)
    assert split_off(full, flen, foff)[lo:hi] == split_off(a, alen, aoff)
