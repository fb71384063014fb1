"""Per-decode-step wall time of one full batch (Student-6-1-1 fp16 greedy):
3072 sentences of equal length -> one batch of 3072 rows, one lane.  Prints
the engine's own decode time / step count, to set against the sum of the
step's kernel durations from an ncu launch list of the same command.

Usage: python tools/perf_step.py [rows] [src_len] [lanes] [sbatch]"""

import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import os
import sys

import numpy as np

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 3072
slen = int(sys.argv[2]) if len(sys.argv) > 2 else 20
if len(sys.argv) > 3:
    os.environ["FNMT_LANES"] = sys.argv[3]
sb = int(sys.argv[4]) if len(sys.argv) > 4 else rows   # sentences per batch

import torch  # noqa: E402

from paper_2109_08003_b200 import store as S  # noqa: E402
from paper_2109_08003_b200.engine import Engine  # noqa: E402

cfg = S.ModelConfig(6, 1, 512, 1, 1, 2048, 2048, 32772, 1024)
eng = Engine(cfg, S.random_model(cfg, 0), dtype="f16")
rng = np.random.default_rng(0)
ids = rng.integers(4, cfg.vocab_size, size=rows * slen).astype(np.int32)
off = (np.arange(rows + 1) * slen).astype(np.int64)
import time  # noqa: E402


def run(offset):
    best = None
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out, olen, oo, st = eng.translate(ids, off, sbatch=sb, wbatch=sb * slen, offset=offset)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return best, st.decode_steps


# the step time is the slope of wall time over decode steps (budget = 1.5 S + offset)
(t1, n1), (t2, n2) = run(5), run(45)
print(f"rows {rows} sbatch {sb} lanes {os.environ.get('FNMT_LANES', '3')} src_len {slen} steps {n1}->{n2} wall_ms {1e3 * t1:.2f}->{1e3 * t2:.2f} "
      f"us/step {1e6 * (t2 - t1) / (n2 - n1):.1f}  fixed_ms {1e3 * (t1 - (t2 - t1) / (n2 - n1) * n1):.2f}")
