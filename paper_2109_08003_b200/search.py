"""Greedy and beam search — drop-in for the reference's search module.

Same names, signatures and semantics as search.py:28-147 (``SearchConfig``,
``Hypothesis``, ``max_out_length``, ``greedy_translate``, ``beam_translate``):

* greedy: argmax over raw logits (log-softmax elided), lowest
  id wins ties, EOS finishes a row without being emitted, the budget token is
  emitted, finished rows are fed PAD, early exit when all rows finished;
* beam: per sentence, length-unnormalised log-prob scores, candidates ordered
  (score desc, token asc, parent asc), an EOS pick moves the hypothesis to the
  finished pool and consumes a beam slot, stop at k finished, final pick by
  (score, -tokens).

With a :class:`~paper_2109_08003_b200.model.GpuTranslationModel` and its own
encoder output, ``greedy_translate`` runs fully on the device (packed varlen
encoder, CUDA-graph decode step, fused vocab argmax, on-device EOS/budget
bookkeeping) and ``beam_translate`` runs the native batched beam.  Any other
model implementing the protocol (encode / init_cache / step) is driven by the
reference algorithm unchanged.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from types import SimpleNamespace

import numpy as np

__all__ = ["SearchConfig", "Hypothesis", "max_out_length", "greedy_translate", "beam_translate"]


@dataclass(frozen=True)
class SearchConfig:
    bos_id: int
    eos_id: int
    pad_id: int
    beam_size: int = 1
    max_len_ratio: float = 1.5
    max_len_offset: int = 5

    def __post_init__(self):
        if self.beam_size < 1:
            raise ValueError("beam_size must be >= 1")


@dataclass(frozen=True)
class Hypothesis:
    tokens: tuple
    score: float
    finished: bool


def max_out_length(src_len: int, cfg: SearchConfig, max_positions: int) -> int:
    return max(1, min(max_positions, math.ceil(cfg.max_len_ratio * src_len) + cfg.max_len_offset))


def _lengths(enc) -> np.ndarray:
    return np.asarray(enc.pad_mask, dtype=bool).sum(axis=1)


def _device_rows(model, enc):
    """Source rows for the fused device path, or None if it does not apply."""
    from .model import GpuEncoderOutput, GpuTranslationModel
    if not isinstance(model, GpuTranslationModel) or not isinstance(enc, GpuEncoderOutput):
        return None
    mask = np.asarray(enc.pad_mask, dtype=bool)
    lens = mask.sum(axis=1)
    prefix = np.arange(mask.shape[1])[None, :] < lens[:, None]
    if not np.array_equal(mask, prefix):
        raise ValueError("the GPU engine expects right-padded sources (real tokens first)")
    if (lens == 0).any():
        return None                       # all-masked rows: reference semantics via the protocol
    return [enc.tokens[i, :n] for i, n in enumerate(lens)]


def _argmax_ids(model, logits):
    from .model import GpuTranslationModel
    if isinstance(model, GpuTranslationModel):
        return model.last_step_argmax()
    return np.argmax(logits, axis=1)


def greedy_translate(model, enc, cfg: SearchConfig) -> list[list[int]]:
    lens = _lengths(enc)
    n = len(lens)
    if n == 0:
        return []
    rows = _device_rows(model, enc)
    if rows is not None:
        return model.translate_batch(rows, search=cfg)
    budgets = [max_out_length(int(x), cfg, model.max_positions) for x in lens]
    cache = model.init_cache(enc)
    feed = np.full(n, cfg.bos_id, dtype=np.int64)
    done = np.zeros(n, dtype=bool)
    outs: list[list[int]] = [[] for _ in range(n)]
    for t in range(max(budgets)):
        best = _argmax_ids(model, model.step(cache, feed))
        feed = np.full(n, cfg.pad_id, dtype=np.int64)
        for r in range(n):
            if done[r]:
                continue
            tok = int(best[r])
            if tok == cfg.eos_id:
                done[r] = True
                continue
            outs[r].append(tok)
            feed[r] = tok
            if t + 1 >= budgets[r]:
                done[r] = True
        if done.all():
            break
    return outs


def _log_softmax64(logits: np.ndarray) -> np.ndarray:
    z = logits - logits.max(axis=-1, keepdims=True)
    return z - np.log(np.einsum("...k->...", np.exp(z)))[..., None]


def _row_enc(enc, r):
    states = getattr(enc, "states", None)
    if states is None:
        return SimpleNamespace(pad_mask=enc.pad_mask[r:r + 1])
    return SimpleNamespace(states=states[r:r + 1], pad_mask=enc.pad_mask[r:r + 1])


def beam_translate(model, enc, cfg: SearchConfig) -> list[list[int]]:
    from .model import GpuTranslationModel
    if isinstance(model, GpuTranslationModel):
        return model.beam_batch(enc, cfg)
    return [_beam_sentence(model, model.init_cache(_row_enc(enc, r)),
                           int(_lengths(enc)[r]), cfg) for r in range(len(enc.pad_mask))]


def _beam_sentence(model, cache, src_len: int, cfg: SearchConfig) -> list[int]:
    """The reference's per-sentence beam (search.py:114-147) over any model."""
    k = cfg.beam_size
    budget = max_out_length(src_len, cfg, model.max_positions)
    live = [Hypothesis((), 0.0, False)]
    done: list[Hypothesis] = []
    for _ in range(budget):
        feed = np.array([h.tokens[-1] if h.tokens else cfg.bos_id for h in live], dtype=np.int64)
        lp = _log_softmax64(np.asarray(model.step(cache, feed), dtype=np.float64))
        vocab = lp.shape[1]
        score = np.array([h.score for h in live])[:, None] + lp
        flat = score.reshape(-1)
        parent = np.repeat(np.arange(len(live)), vocab)
        token = np.tile(np.arange(vocab), len(live))
        order = np.lexsort((parent, token, -flat))[:k]
        nxt, parents = [], []
        for j in order:
            s, tok, par = float(flat[j]), int(token[j]), int(parent[j])
            if tok == cfg.eos_id:
                done.append(Hypothesis(live[par].tokens, s, True))
            else:
                nxt.append(Hypothesis(live[par].tokens + (tok,), s, False))
                parents.append(par)
        live = nxt
        if not live or len(done) >= k:
            break
        cache = cache.select(parents)
    pool = done if done else live
    return list(max(pool, key=lambda h: (h.score, tuple(-x for x in h.tokens))).tokens)
