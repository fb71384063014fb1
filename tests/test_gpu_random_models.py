"""Acceptance-scale randomized equivalence (reference
tests/test_acceptance.py:163-216, shapes from its _student_shape_pool and
tests/helpers.py:47-62): >= 100 random student-shaped models, each with
random norm variant / embedding sharing / seed.

Per model, on the GPU engine:
  * fp32 parity mode: every incremental decode_step's logits within 1e-4 of
    the oracle (the reference's cached-vs-recompute check is 1e-5 on the
    reference itself; the north-star GPU tolerance is 1e-4), token-for-token
    identical greedy steps, and the fused corpus decode (graph + argmax
    epilogue) identical to the oracle's greedy;
  * fp16: the same steps' logits within 1e-2.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import nmt_oracle as O  # noqa: E402
from paper_2109_08003_b200 import store as S  # noqa: E402
from paper_2109_08003_b200.model import GpuTranslationModel  # noqa: E402


def shape_pool(d):
    # (n_enc, n_dec, heads_enc, heads_dec, ffn_dec) — test_acceptance.py:148-160
    return [(12, 1, 8, 1, d), (6, 1, 8, 1, d), (6, 1, 8, 1, 0), (3, 1, 8, 1, d),
            (6, 6, 8, 8, 4 * d), (6, 1, 8, 8, 4 * d), (6, 1, 1, 1, 4 * d)]


def models(n=100, seed=2024):
    rng = np.random.default_rng(seed)
    for i in range(n):
        d = int(rng.choice([32, 64]))
        ne, nd, he, hd, fd = shape_pool(d)[i % 7]
        cfg = S.ModelConfig(n_enc_layers=ne, n_dec_layers=nd, d_model=d, n_heads_enc=he,
                            n_heads_dec=hd, ffn_dim_enc=4 * d, ffn_dim_dec=fd, vocab_size=48,
                            max_positions=64, norm_variant=str(rng.choice(["l2", "l1"])),
                            shared_embeddings=bool(rng.integers(0, 2)))
        wseed = int(rng.integers(0, 2 ** 31))
        rows = [rng.integers(4, 48, size=int(rng.integers(3, 7))).astype(np.int64)
                for _ in range(2)]
        yield i, cfg, wseed, rows


def test_incremental_decode_on_100_random_models():
    checked = 0
    worst32 = worst16 = 0.0
    for i, cfg, wseed, rows in models():
        a = O.arch_of(cfg)
        p = O.make_params(a, wseed)
        w = S.random_model(cfg, wseed)
        tok, valid = O.pad_rows(rows)
        want_greedy = O.greedy(a, p, tok, valid)
        budgets = [O.out_budget(len(r), cfg.max_positions) for r in rows]
        for dtype, tol in (("f32", 1e-4), ("f16", 1e-2)):
            m = GpuTranslationModel(cfg, w, dtype=dtype)
            cache = m.init_cache(m.encode(tok, valid))
            oc = O.start_cache(a, p, O.encoder(a, p, tok, valid), valid)
            prev = np.full(2, 2, np.int64)
            done = [False, False]
            for t in range(max(budgets)):
                want = O.decoder_step(a, p, oc, prev)
                got = m.step(cache, prev)
                err = float(np.abs(got - want).max() / max(1.0, np.abs(want).max()))
                assert err <= tol, (i, dtype, t, err, cfg)
                if dtype == "f32":
                    worst32 = max(worst32, err)
                    assert np.array_equal(got.argmax(axis=1), want.argmax(axis=1)), (i, t)
                else:
                    worst16 = max(worst16, err)
                nxt = want.argmax(axis=1)
                prev = np.zeros(2, np.int64)
                for b in range(2):
                    if done[b]:
                        continue
                    if nxt[b] == 3 or t + 1 >= budgets[b]:
                        done[b] = True
                    else:
                        prev[b] = nxt[b]
                if all(done):
                    break
            if dtype == "f32":
                assert m.translate_batch(rows) == want_greedy, (i, cfg)
        checked += 1
    print(f"{checked} models: worst f32 logits rel err {worst32:.2e}, f16 {worst16:.2e}")
    assert checked >= 100
