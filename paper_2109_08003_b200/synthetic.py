"""Synthetic workloads of BASELINE.json / SURVEY.md §8(d).

* newstest-shaped corpus: source length clip(round(Gamma(k=3, theta=8)), 1, 200)
  (mean ~24 BPE tokens, p99 ~67; the paper's 18-word average at ~1.33 BPE
  tokens/word), ids uniform in [4, vocab), no BOS/EOS appended.
* config 1: 64 sentences, lengths uniform in [10, 40].
"""

from __future__ import annotations

import numpy as np


def newstest_lengths(n: int, seed: int = 20211) -> np.ndarray:
    g = np.random.default_rng(seed)
    return np.clip(np.rint(g.gamma(3.0, 8.0, size=n)), 1, 200).astype(np.int32)


def newstest_corpus(n: int, vocab: int, seed: int = 20211):
    """(ids int32 flat, offsets int64 [n+1], lengths int32 [n])."""
    lengths = newstest_lengths(n, seed)
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lengths, out=offsets[1:])
    ids = np.random.default_rng(seed + 1).integers(4, vocab, size=int(offsets[-1]),
                                                   dtype=np.int32)
    return ids, offsets, lengths


def config1_rows(n: int = 64, seed: int = 1234, vocab: int = 32772):
    g = np.random.default_rng(seed)
    lens = g.integers(10, 41, size=n)
    return [g.integers(4, vocab, size=int(L)).astype(np.int64) for L in lens]
