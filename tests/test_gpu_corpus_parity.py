"""Parity on the BENCHMARKED workload (BASELINE.json configs 2-5).

The sentences are sampled from chunk 0 of the 2^20-sentence newstest-shaped
corpus (one bench step) and translated IN THEIR REAL BATCHES: the whole chunk
(or, for beam, its first 8192 sentences) goes through the production engine
call with the bench's caps (sbatch/wbatch 3072/64000), the default concurrent
decode lanes, folded cross attention (single-head decoders) and PDL — the
code path bench.py times.  The reference outputs and per-step near-tie data
come from tests/golden/corpus_*.npz (oracle/make_golden_corpus.py ran the
unmodified reference on the same sentences).

Bar (BASELINE.json north_star): token-identical on >= 99% of sentences and
every divergence a near-tie (tests/parity.py: reference top-1 vs the
engine's pick within 0.05 logits for fp16, 0.10 for bf16; beam: the same in
summed log-probs at the first step the engine's hypothesis leaves the
reference beam).  Also the production-vocab (V = 32772) fp16 logits of the
students' decode_step within 1e-2 of the oracle.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import nmt_oracle as O  # noqa: E402
from paper_2109_08003_b200 import store as S  # noqa: E402
from paper_2109_08003_b200.engine import Engine, budgets_of  # noqa: E402
from paper_2109_08003_b200.model import GpuTranslationModel  # noqa: E402
from paper_2109_08003_b200.synthetic import newstest_corpus  # noqa: E402
from oracle import parity as P  # noqa: E402

CHUNK = 65536
BASE = dict(n_enc_layers=6, n_dec_layers=1, d_model=512, n_heads_enc=1, n_heads_dec=1,
            ffn_dim_enc=2048, ffn_dim_dec=2048, vocab_size=32772, max_positions=1024)
MODELS = {
    "s611": BASE,
    "s618": dict(BASE, n_heads_enc=8, n_heads_dec=8),
    "s668_beam4": dict(BASE, n_dec_layers=6, n_heads_enc=8, n_heads_dec=8,
                       shared_embeddings=False),
    "deep_beam4": dict(BASE, n_enc_layers=12, n_dec_layers=6, d_model=768, n_heads_enc=8,
                       n_heads_dec=8, ffn_dim_enc=3072, ffn_dim_dec=3072),
}


@pytest.fixture(scope="module")
def corpus():
    return newstest_corpus(1 << 20, 32772)


def translate_slice(eng, corpus, n, beam=1):
    ids, off, _ = corpus
    out, olen, oof, _ = eng.translate(ids, off[:n + 1], sbatch=3072, wbatch=64000, beam=beam)
    return out, olen, oof


def rows_at(out, olen, oof, idx):
    return [out[oof[i]:oof[i] + olen[i]].tolist() for i in idx]


@pytest.mark.parametrize("tag", ["s611", "s618"])
def test_greedy_corpus_chunk_fp16(golden, corpus, tag):
    """Configs 2 / 3: Student-6-1-1 / 6-1-8 fp16 greedy on corpus chunk 0."""
    fx = golden(f"corpus_{tag}")
    cfg = S.ModelConfig(**MODELS[tag])
    eng = Engine(cfg, S.random_model(cfg, 0), dtype="f16")
    out, olen, oof = translate_slice(eng, corpus, CHUNK)
    rep = P.greedy_report(rows_at(out, olen, oof, fx["idx"]), fx)
    print(tag, "fp16 greedy parity:", rep)
    assert rep["pass"], rep


@pytest.mark.parametrize("tag,dtype", [("s668_beam4", "f16"), ("deep_beam4", "bf16")])
def test_beam_corpus_slice(golden, corpus, tag, dtype):
    """Configs 4 / 5: Student-6-6-8 fp16 and Deep-12-768 bf16, beam 4."""
    fx = golden(f"corpus_{tag}")
    cfg = S.ModelConfig(**MODELS[tag])
    eng = Engine(cfg, S.random_model(cfg, 0), dtype=dtype)
    out, olen, oof = translate_slice(eng, corpus, 8192, beam=int(fx["k"]))
    _, off, lengths = corpus
    budgets = budgets_of(lengths[fx["idx"]], 1.5, 5, cfg.max_positions)
    tie = P.NEAR_TIE if dtype == "f16" else P.NEAR_TIE_BF16
    rep = P.beam_report(rows_at(out, olen, oof, fx["idx"]), fx, budgets, near_tie=tie)
    print(tag, dtype, "beam parity:", rep)
    assert rep["pass"], rep


@pytest.mark.parametrize("tag", ["s611", "s618"])
def test_production_vocab_logits_fp16(corpus, tag):
    """decode_step at d = 512, V = 32772 (model.py:308-344): fp16 logits of 6
    forced steps on 8 corpus sentences within 1e-2 of the oracle, measured as
    max|got - want| / max(1, max|want|) (test_gpu_parity.rel_err)."""
    ids, off, _ = corpus
    cfg = S.ModelConfig(**MODELS[tag])
    a = O.arch_of(cfg)
    p = O.make_params(a, 0)
    rows = [ids[off[i]:off[i + 1]].astype(np.int64) for i in range(100, 108)]
    tok, valid = O.pad_rows(rows)
    m = GpuTranslationModel(cfg, S.random_model(cfg, 0), dtype="f16")
    cache = m.init_cache(m.encode(tok, valid))
    oc = O.start_cache(a, p, O.encoder(a, p, tok, valid), valid)
    prev = np.full(len(rows), 2, np.int64)
    worst = 0.0
    for t in range(6):
        want = O.decoder_step(a, p, oc, prev)
        got = m.step(cache, prev)
        err = float(np.abs(got - want).max() / max(1.0, np.abs(want).max()))
        worst = max(worst, err)
        assert err <= 1e-2, (t, err)
        prev = want.argmax(axis=1).astype(np.int64)
    print(tag, "worst fp16 logits rel err", worst)


WIDE_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2109_08003_b200 import store as S
from paper_2109_08003_b200.engine import Engine
from paper_2109_08003_b200.synthetic import newstest_corpus
ids, off, _ = newstest_corpus(1 << 20, 32772)
cfg = S.ModelConfig(6, 1, 512, 8, 8, 2048, 2048, 32772, 1024)
eng = Engine(cfg, S.random_model(cfg, 0), dtype="f16")
out, olen, oof, _ = eng.translate(ids, off[:65536 + 1], sbatch=3072, wbatch=64000)
np.savez(sys.argv[2], out=out, olen=olen, oof=oof)
"""


@pytest.mark.parametrize("mh_tables", ["0", "1"])
def test_greedy_corpus_wide_s618(golden, tmp_path, mh_tables):
    """Config 3 on a wider, disjoint sample (2048 sentences of chunk 0,
    corpus_s618_wide.npz), with and without the multi-head layer-0 step tables
    (FNMT_STEP_TABLES_MH, a process-wide switch: each variant runs in its own
    process): both at the north-star bar."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    fx = golden("corpus_s618_wide")
    f = tmp_path / f"wide_{mh_tables}.npz"
    env = dict(os.environ, FNMT_STEP_TABLES_MH=mh_tables)
    root = Path(__file__).resolve().parent.parent
    r = subprocess.run([sys.executable, "-c", WIDE_SCRIPT, str(root), str(f)], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    d = np.load(f)
    rep = P.greedy_report(rows_at(d["out"], d["olen"], d["oof"], fx["idx"]), fx)
    print("s618_wide mh_tables", mh_tables, "fp16 greedy parity:",
          {k: rep[k] for k in ("sentences", "identical", "identical_frac", "all_near_ties")})
    assert rep["pass"], rep
