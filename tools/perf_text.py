"""Text-level throughput of the Translator facade (tokenize -> BPE -> ids ->
engine -> detokenize) for Student-6-1-1 fp16 on a synthetic corpus: lines of
newstest-shaped length whose words are Zipf-distributed vocabulary tokens.

Usage: python tools/perf_text.py [n_lines] [workers]"""

import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import sys

import numpy as np

from paper_2109_08003_b200 import store as S
from paper_2109_08003_b200.synthetic import newstest_corpus
from paper_2109_08003_b200.textpipe import synthetic_vocabulary
from paper_2109_08003_b200.translator import RunConfig, Translator


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
    workers = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    cfg = S.ModelConfig(6, 1, 512, 1, 1, 2048, 2048, 32772, 1024)
    vocab = synthetic_vocabulary(cfg.vocab_size)
    toks = vocab.all_tokens()[4:]
    rng = np.random.default_rng(0)
    _, _, lengths = newstest_corpus(n, cfg.vocab_size)
    ranks = np.minimum(rng.zipf(1.2, size=int(lengths.sum())), len(toks)) - 1
    lines, o = [], 0
    for L in lengths:
        lines.append(" ".join(toks[r] for r in ranks[o:o + L]))
        o += int(L)
    tr = Translator(cfg, S.random_model(cfg, 0), vocab,
                    run=RunConfig(precision="f16", workers=workers, chunk_lines=8192))
    tr.translate_lines(lines[:20000])
    for _ in range(2):
        rep = tr.bench(lines)
        print({k: (round(v) if isinstance(v, float) and v > 100 else v) for k, v in rep.items()})


if __name__ == "__main__":   # text workers come from a forkserver (re-imports __main__)
    main()
