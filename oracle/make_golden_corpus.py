"""Golden fixtures for parity ON THE BENCHMARKED WORKLOAD (test infrastructure).

BASELINE.json configs 2-5 translate the 2^20-sentence newstest-shaped corpus
(paper_2109_08003_b200/synthetic.py, seed 20211).  This script samples
sentences from corpus chunk 0 (the first 65 536 sentences, one bench step) and
records what the UNMODIFIED reference does with them, so the GPU tests and the
bench can compare the engine's output for the same sentences, translated in
their real batches (caps 3072/64000, default lanes), against it:

* greedy (Student-6-1-1, Student-6-1-8; random_model seed 0): the reference's
  ``search.greedy_translate`` (search.py:58-86) through a recording wrapper of
  ``TranslationModel.step`` that keeps, for every live step of every row, the
  top-1 / top-2 logits and the runner-up id (the near-tie report);
* beam 4 (Student-6-6-8 unshared, Deep-12-768): ``oracle.beam_sentence`` with
  its candidate trace (per step the first 3k candidates in the reference's
  sort order, search.py:121-127), cross-checked against the reference's own
  ``search.beam_translate`` output for every sentence (must be identical).

Writes tests/golden/corpus_<tag>.npz.  Runs the reference from
/root/reference (build container only); the fixtures travel, the reference
does not.  Work is spread over the host cores with one process per core
(OMP_NUM_THREADS=1; the reference's einsum is batch-invariant, so the
grouping does not change any value).

Usage: python oracle/make_golden_corpus.py [greedy|beam|all|greedy_wide]
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

import numpy as np

os.environ.setdefault("OMP_NUM_THREADS", "1")
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(HERE.parent))
from make_golden import OUT, STUDENTS, import_reference, padded  # noqa: E402

CORPUS = 1 << 20
CHUNK = 65536

# (tag, STUDENTS key, beam, sample indices inside chunk 0)
GREEDY = [("s611", "student_6_1_1", np.arange(1024) * 64),
          ("s618", "student_6_1_8", np.arange(512) * 128 + 17)]
# a wider Student-6-1-8 sample (2048 sentences, disjoint from s618) for the
# multi-head step-table decision (tests/test_gpu_corpus_parity.py)
GREEDY_WIDE = [("s618_wide", "student_6_1_8", np.arange(2048) * 32 + 3)]
BEAM = [("s668_beam4", "student_6_6_8", np.arange(32) * 256 + 5),
        ("deep_beam4", "deep_12_768", np.arange(24) * 341 + 9)]
BEAM_K = 4

_S = {}


def corpus():
    from paper_2109_08003_b200.synthetic import newstest_corpus
    ids, off, _ = newstest_corpus(CORPUS, 32772)
    return ids, off


class Recorder:
    """TranslationModel protocol wrapper recording per-step top-2 logits."""

    def __init__(self, tm):
        self.tm = tm
        self.max_positions = tm.max_positions
        self.top = []

    def init_cache(self, enc):
        return self.tm.init_cache(enc)

    def step(self, cache, prev):
        lg = self.tm.step(cache, prev)
        i1 = np.argmax(lg, axis=1)
        rows = np.arange(lg.shape[0])
        v1 = lg[rows, i1].copy()
        tmp = lg.copy()
        tmp[rows, i1] = -np.inf
        i2 = np.argmax(tmp, axis=1)
        self.top.append((v1, tmp[rows, i2].copy(), i2.astype(np.int32)))
        return lg


def _greedy_worker(rows):
    ref, tm = _S["ref"], _S["tm"]
    S = ref.search
    tok, valid = padded(rows)
    rec = Recorder(tm)
    enc = tm.encode(tok, valid)
    outs = S.greedy_translate(rec, enc, S.SearchConfig(bos_id=2, eos_id=3, pad_id=0))
    res = []
    for r, o in enumerate(outs):
        budget = S.max_out_length(len(rows[r]), S.SearchConfig(bos_id=2, eos_id=3, pad_id=0),
                                  tm.max_positions)
        n_live = min(budget, len(o) + 1, len(rec.top))   # steps the row was live
        v1 = np.array([rec.top[t][0][r] for t in range(n_live)], np.float32)
        v2 = np.array([rec.top[t][1][r] for t in range(n_live)], np.float32)
        i2 = np.array([rec.top[t][2][r] for t in range(n_live)], np.int32)
        res.append((o, v1, v2, i2))
    return res


def _beam_worker(job):
    from oracle import nmt_oracle as O
    i, row = job
    ref, tm, a, p = _S["ref"], _S["tm"], _S["arch"], _S["params"]
    S = ref.search
    tok, valid = padded([row])
    states = O.encoder(a, p, tok, valid)
    trace = []
    hyp, score, fin = O.beam_sentence(a, p, states, valid, BEAM_K, trace=trace)
    enc = tm.encode(tok, valid)
    want = S.beam_translate(tm, enc, S.SearchConfig(bos_id=2, eos_id=3, pad_id=0,
                                                    beam_size=BEAM_K))[0]
    if list(hyp) != list(want):
        raise SystemExit(f"oracle beam differs from the reference on sentence {i}")
    return list(hyp), trace


def _setup(key, with_oracle=False):
    ref = import_reference()
    cfg = ref.model.ModelConfig(**STUDENTS[key])
    w = ref.store.random_model(cfg, 0)
    _S["ref"] = ref
    _S["tm"] = ref.model.TranslationModel(cfg, w)
    if with_oracle:
        from oracle import nmt_oracle as O
        a = O.arch_of(cfg)
        _S["arch"] = a
        _S["params"] = O.params_from_weights(a, w)


def run_greedy(procs, sets=GREEDY):
    ids, off = corpus()
    for tag, key, idx in sets:
        t0 = time.time()
        _setup(key)
        rows = [ids[off[i]:off[i + 1]].astype(np.int64) for i in idx]
        groups = [rows[j:j + 8] for j in range(0, len(rows), 8)]
        with mp.get_context("fork").Pool(procs) as pool:
            res = [r for part in pool.map(_greedy_worker, groups, chunksize=1) for r in part]
        out = {"idx": idx.astype(np.int64),
               "out_ids": np.array([t for r in res for t in r[0]], np.int32),
               "out_lens": np.array([len(r[0]) for r in res], np.int32),
               "step_counts": np.array([len(r[1]) for r in res], np.int32),
               "top1": np.concatenate([r[1] for r in res]),
               "top2": np.concatenate([r[2] for r in res]),
               "top2_id": np.concatenate([r[3] for r in res])}
        np.savez_compressed(OUT / f"corpus_{tag}.npz", **out)
        print(f"{tag}: {len(rows)} sentences, {int(out['out_lens'].sum())} words, "
              f"{time.time() - t0:.0f}s", file=sys.stderr)


def run_beam(procs):
    ids, off = corpus()
    for tag, key, idx in BEAM:
        t0 = time.time()
        _setup(key, with_oracle=True)
        jobs = [(int(i), ids[off[i]:off[i + 1]].astype(np.int64)) for i in idx]
        with mp.get_context("fork").Pool(procs) as pool:
            res = pool.map(_beam_worker, jobs, chunksize=1)
        steps = [len(tr) for _, tr in res]
        out = {"idx": idx.astype(np.int64), "k": np.array(BEAM_K),
               "out_ids": np.array([t for h, _ in res for t in h], np.int32),
               "out_lens": np.array([len(h) for h, _ in res], np.int32),
               "step_counts": np.array(steps, np.int32),
               "cand_score": np.concatenate([np.stack([s for s, _, _ in tr]) for _, tr in res]),
               "cand_tok": np.concatenate([np.stack([t for _, t, _ in tr]) for _, tr in res]),
               "cand_par": np.concatenate([np.stack([q for _, _, q in tr]) for _, tr in res])}
        np.savez_compressed(OUT / f"corpus_{tag}.npz", **out)
        print(f"{tag}: {len(jobs)} sentences, {int(out['out_lens'].sum())} words, "
              f"{time.time() - t0:.0f}s", file=sys.stderr)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    procs = os.cpu_count() or 1
    if what in ("greedy", "all"):
        run_greedy(procs)
    if what == "greedy_wide":
        run_greedy(procs, GREEDY_WIDE)
    if what in ("beam", "all"):
        run_beam(procs)
