"""Per-decode-step wall time of one full batch (Student-6-1-1 fp16 greedy):
3072 sentences of equal length -> one batch of 3072 rows, one lane.  Prints
the engine's own decode time / step count, to set against the sum of the
step's kernel durations from an ncu launch list of the same command.

Usage: python -m paper_2109_08003_b200.perf_step [rows] [src_len] [lanes]"""
import os
import sys

import numpy as np

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 3072
slen = int(sys.argv[2]) if len(sys.argv) > 2 else 20
if len(sys.argv) > 3:
    os.environ["FNMT_LANES"] = sys.argv[3]

import torch  # noqa: E402

from paper_2109_08003_b200 import store as S  # noqa: E402
from paper_2109_08003_b200.engine import Engine  # noqa: E402

cfg = S.ModelConfig(6, 1, 512, 1, 1, 2048, 2048, 32772, 1024)
eng = Engine(cfg, S.random_model(cfg, 0), dtype="f16")
rng = np.random.default_rng(0)
ids = rng.integers(4, cfg.vocab_size, size=rows * slen).astype(np.int32)
off = (np.arange(rows + 1) * slen).astype(np.int64)
for i in range(3):
    out, olen, oo, st = eng.translate(ids, off, sbatch=rows, wbatch=rows * slen)
    torch.cuda.synchronize()
    print(f"rows {rows} src_len {slen} batches {st.batches} steps {st.decode_steps} "
          f"encode_ms {st.encode_ms:.3f} decode_ms {st.decode_ms:.3f} "
          f"us/step {1e3 * st.decode_ms / max(st.decode_steps, 1):.1f} launches {st.gpu_launches}")
