"""Golden beam-search outputs from the UNMODIFIED reference on student-shaped
models (test infrastructure; see make_golden.py for the import shim).

Writes tests/golden/beam_students.npz: for Student-6-1-1 and Student-6-1-8
(random_model seed 0) and beam sizes 2 and 4, the reference's beam_translate
output for the first N sentences of config 1, plus every candidate score gap
needed for the near-tie report (best vs runner-up final scores).
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent))
from make_golden import OUT, STUDENTS, import_reference, padded  # noqa: E402


def main(n_sent: int = 4):
    ref = import_reference()
    M, S = ref.model, ref.search
    g = np.random.default_rng(1234)
    lens = g.integers(10, 41, size=64)
    rows = [g.integers(4, 32772, size=int(L)).astype(np.int64) for L in lens][:n_sent]
    out = {"src_ids": np.concatenate(rows), "src_lens": np.array([len(r) for r in rows])}
    for tag in ("student_6_1_1", "student_6_1_8"):
        cfg = M.ModelConfig(**STUDENTS[tag])
        tm = M.TranslationModel(cfg, ref.store.random_model(cfg, 0))
        tok, valid = padded(rows)
        enc = tm.encode(tok, valid)
        for k in (2, 4):
            t0 = time.time()
            res = S.beam_translate(tm, enc, S.SearchConfig(bos_id=2, eos_id=3, pad_id=0,
                                                           beam_size=k))
            print(f"{tag} beam{k}: {time.time() - t0:.1f}s", file=sys.stderr)
            out[f"{tag}_beam{k}_ids"] = np.array([t for r in res for t in r], np.int64)
            out[f"{tag}_beam{k}_lens"] = np.array([len(r) for r in res], np.int64)
    np.savez_compressed(OUT / "beam_students.npz", **out)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
