"""Live per-launch durations of one decode batch (engine profiler: every
launch bracketed by CUDA events on the engine stream, un-captured), Student-6-1-1
fp16 greedy, ROWS equal-length sentences in one batch.  Prints the median
duration of each launch position within a decode step.

Usage: python tools/step_live.py [rows] [src_len]"""

import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2109_08003_b200 import _capi  # noqa: E402
from paper_2109_08003_b200 import store as S  # noqa: E402
from paper_2109_08003_b200.engine import Engine  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 3072
slen = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = S.ModelConfig(6, 1, 512, 1, 1, 2048, 2048, 32772, 1024)
eng = Engine(cfg, S.random_model(cfg, 0), dtype="f16")
rng = np.random.default_rng(0)
ids = rng.integers(4, cfg.vocab_size, size=rows * slen).astype(np.int32)
off = (np.arange(rows + 1) * slen).astype(np.int64)
eng.translate(ids, off, sbatch=rows, wbatch=rows * slen)
eng.profile(True)
eng.translate(ids, off, sbatch=rows, wbatch=rows * slen)
torch.cuda.synchronize()
log = eng.profile_log()
names = _capi.KERNEL_CLASSES
cls, ms = log["cls"], log["ms"]
search = names.index("search")
# decode steps end with the search-class launch (greedy update + next embedding)
ends = np.nonzero(cls == search)[0]
per = np.diff(ends)
L = int(np.bincount(per).argmax())
steps = [ms[e - L + 1:e + 1] for e, p in zip(ends[1:], per) if p == L]
pos_cls = [names[c] for c in cls[ends[1] - L + 1:ends[1] + 1]]
med = np.median(np.array(steps), axis=0)
print(f"rows {rows} src_len {slen}: {len(steps)} steps of {L} launches, "
      f"sum of medians {1e3 * med.sum():.1f} us")
for c, m in zip(pos_cls, med):
    print(f"  {c:14s} {1e3 * m:8.1f} us")
