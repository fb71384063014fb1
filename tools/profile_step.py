"""Small fixed workload for ncu: one corpus slice through the engine
(Student-6-1-1, fp16 greedy by default).

Usage: python tools/profile_step.py [n_sentences] [dtype] [beam]"""

import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2109_08003_b200 import store as S  # noqa: E402
from paper_2109_08003_b200.engine import Engine  # noqa: E402
from paper_2109_08003_b200.synthetic import newstest_corpus  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
cfg = S.ModelConfig(6, 1, 512, 1, 1, 2048, 2048, 32772, 1024)
ids, off, lens = newstest_corpus(n, cfg.vocab_size)
eng = Engine(cfg, S.random_model(cfg, 0), dtype=sys.argv[2] if len(sys.argv) > 2 else "f16")
beam = int(sys.argv[3]) if len(sys.argv) > 3 else 1
for _ in range(2):
    out, olen, oo, st = eng.translate(ids, off, sbatch=3072, wbatch=64000, beam=beam)
torch.cuda.synchronize()
print("words", int(olen.sum()), "launches", st.gpu_launches, "batches", st.batches,
      "steps", st.decode_steps, "ms", st.total_ms)
