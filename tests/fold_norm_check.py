"""Subprocess body of test_fold_norm_path (FNMT_FOLD_NORM=1 is read once):
Student-6-1-1 fp16 with residual + norm2 inside the folded cross attention,
BASELINE config 1 (64 sentences) against the reference's recorded greedy ids."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import nmt_oracle as O  # noqa: E402
from paper_2109_08003_b200 import store as S  # noqa: E402
from paper_2109_08003_b200.engine import Engine  # noqa: E402


def main():
    g = np.load(ROOT / "tests" / "golden" / "config1_greedy.npz")
    want, o = [], 0
    for n in g["out_lens"]:
        want.append([int(x) for x in g["out_ids"][o:o + n]])
        o += int(n)
    cfg = S.ModelConfig(6, 1, 512, 1, 1, 2048, 2048, 32772, 1024)
    eng = Engine(cfg, S.random_model(cfg, 0), dtype="f16")
    rows = O.config1_sentences()
    lengths = np.array([len(r) for r in rows])
    offsets = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    out, olen, off, _ = eng.translate(np.concatenate(rows).astype(np.int32), offsets,
                                      sbatch=128, wbatch=2048)
    got = [out[a:a + n].tolist() for a, n in zip(off, olen)]
    same = sum(x == y for x, y in zip(got, want))
    assert same >= 63, same
    print("fold norm ok", same)


if __name__ == "__main__":
    main()
