"""Debug probe: translate each 65536-sentence chunk of the bench corpus
through Engine.translate_device (as bench.py does) and report progress, to
find chunks that fail.  Usage: python tools/chunk_probe.py [first last]"""

import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import sys

import numpy as np
import torch

from paper_2109_08003_b200 import store as S
from paper_2109_08003_b200.engine import Engine, budgets_of
from paper_2109_08003_b200.synthetic import newstest_corpus

first = int(sys.argv[1]) if len(sys.argv) > 1 else 0
last = int(sys.argv[2]) if len(sys.argv) > 2 else 15
cfg = S.ModelConfig(6, 1, 512, 1, 1, 2048, 2048, 32772, 1024)
ids, offsets, lengths = newstest_corpus(1 << 20, cfg.vocab_size)
eng = Engine(cfg, S.random_model(cfg, 0), dtype="f16")
eng.reserve(3072, 64000)
dev = torch.device("cuda", 0)
d_ids = torch.from_numpy(ids).to(dev)
d_off = torch.from_numpy(offsets).to(dev)
C = 65536
for c in range(first, last + 1):
    lo, hi = c * C, (c + 1) * C
    L = lengths[lo:hi]
    b = budgets_of(L, 1.5, 5, cfg.max_positions)
    off = np.zeros(len(b), np.int64)
    np.cumsum(b[:-1], out=off[1:])
    d_out = torch.empty(int(b.sum()), dtype=torch.int32, device=dev)
    d_len = torch.empty(len(L), dtype=torch.int32, device=dev)
    print("chunk", c, "max len", int(L.max()), "out", int(b.sum()), flush=True)
    st = eng.translate_device(d_ids, d_off[lo:hi + 1], L, d_out, off, torch.from_numpy(off).to(dev),
                              d_len)
    torch.cuda.synchronize()
    print("  ok words", int(d_len.sum().item()), "batches", st.batches, flush=True)
