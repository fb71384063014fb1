"""``Translator`` / ``RunConfig``: the reference's text-level translate and
bench entry points on the B200 engine.

The reference ``fastnmt.engine`` module is missing upstream;
its contract is reconstructed from its callers — ``cli.py:34-89``,
``tests/test_engine_cli.py:21-145``, ``tests/test_acceptance.py:408-455``
and SPEC.md:593-650:

* ``Translator(cfg, weights, vocab, codec=None, run=RunConfig())``,
  ``Translator.from_file(path, run=, bpe_codes=)``, ``.codec`` assignable;
* ``translate_lines(lines)``: tokenize -> BPE -> id-map -> (sort/batch ->
  decode on the GPU) -> id-unmap -> BPE-join -> detokenize; line count
  preserved, empty line -> empty line, over-long lines hard-split at
  ``min(1024, max_positions)`` subword tokens and rejoined;
* ``bench(lines)``: ``words_per_second`` = source words / wall seconds plus
  the configured limits, and the GPU-side target-word rate;
* ``selftest()``: the dirty-data / empty / over-long battery.

B200 design: the text stages are host work on ``run.workers`` threads, the
GPU stage is one native ``fnmt_engine_translate`` call per group of chunks
(length-sorted token-budget batching, graph-captured decode, order restore
inside the call).  The three stages are pipelined — chunk i+1 is tokenized
and chunk i-1 detokenized while the engine call for chunk i runs (ctypes
releases the GIL for the native call).  Because every engine kernel is
batch-invariant, the output does not depend on ``workers``,
``chunk_lines``, ``sbatch`` or ``wbatch`` (the reference's worker- and
cap-invariance contracts, test_engine_cli.py:39-55).
"""

from __future__ import annotations

import multiprocessing as mp
import time
from concurrent.futures import ProcessPoolExecutor, ThreadPoolExecutor
from dataclasses import dataclass, replace
from typing import Optional, Sequence

import numpy as np

from . import modelfile
from .store import ModelConfig, config_of
from .textpipe import (BOS_ID, EOS_ID, PAD_ID, BpeCodec, ChunkFailure, Vocabulary, bpe_decode,
                       bpe_encode, clean_line, detokenize, tokenize_word)

_WORD_CACHE_MAX = 1 << 20

PRECISIONS = ("f32", "f16", "bf16", "int8")
HARD_SPLIT = 1024            # SPEC.md:369 default hard limit (BPE tokens)
GPU_GROUP_LINES = 65536      # lines per engine call when the result is batch-invariant


@dataclass(frozen=True)
class RunConfig:
    """Run flags (cli.py:20-45).  Defaults are the paper's GPU decoding
    configuration (sbatch/wbatch 3072/64000) and the fp16
    production precision; ``precision="f32"`` is the bit-faithful parity mode
    and ``"int8"`` the per-column quantized GEMM path (quant8.py)."""

    precision: str = "f16"
    sbatch: int = 3072
    wbatch: int = 64000
    workers: int = 1
    chunk_lines: int = 2000
    beam: int = 1
    pretokenized: bool = False
    max_len_ratio: float = 1.5
    max_len_offset: int = 5
    devices: tuple = (0,)           # GPUs (one engine each; chunk groups round-robin)

    def __post_init__(self):
        if self.precision not in PRECISIONS:
            raise ValueError(f"unknown precision {self.precision!r}")
        for name in ("sbatch", "wbatch", "workers", "chunk_lines", "beam"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be >= 1")
        if self.beam > 8:
            # the engine's corpus path keeps beam state in the fused top-K vocab
            # epilogue (up to 8 candidates per row); GpuTranslationModel's
            # protocol-level beam_translate has no cap
            raise ValueError(f"beam={self.beam}: the GPU Translator supports beam sizes 1-8")
        if not self.devices or any(int(d) < 0 for d in self.devices):
            raise ValueError("devices must list at least one CUDA ordinal")
        object.__setattr__(self, "devices", tuple(int(d) for d in self.devices))


# Text stages in worker processes (run.workers > 1): pure-Python tokenize /
# BPE / detokenize are GIL-bound, so threads do not scale.  The workers come
# from a "forkserver" context — a clean server process that never touched
# CUDA or the engine's lane threads (forking the multi-threaded,
# CUDA-initialised translator process itself is unsafe) — and receive a
# pickled copy of the text stage (vocabulary, codec, split limit) once, in
# their initializer.
_WORKER_STAGE = None


def _init_worker(stage):
    global _WORKER_STAGE
    _WORKER_STAGE = stage


def _proc_ready(_):
    return True


def _proc_to_ids(lines, pretok):
    return _WORKER_STAGE.to_ids(lines, pretok)


def _proc_to_text(chunk, outs, pretok):
    return _WORKER_STAGE.to_text(chunk, outs, pretok)


@dataclass
class _Chunk:
    pieces: list          # list[np.ndarray int32] subword ids, each <= limit
    owner: list           # piece -> line index within the chunk
    n_lines: int


class _TextStage:
    """Host text stages of one (vocabulary, codec, split limit): word-memoised
    tokenize -> BPE -> ids and ids -> BPE-join -> detokenize, plus the worker
    pools that run them.  ``Translator.with_run`` copies share their stage
    (same codec, same pools); assigning ``Translator.codec`` gives that
    translator a fresh stage and leaves the others' pools alone.  Pools close
    when the last translator holding the stage goes away."""

    def __init__(self, vocab: Vocabulary, codec: Optional[BpeCodec], limit: int):
        self.vocab = vocab
        self.codec = codec
        self.limit = limit
        self.word_ids = {False: {}, True: {}}   # per pretokenized flag: word -> ids
        self.pools: dict = {}                   # workers -> process pool

    def __getstate__(self):   # what a worker receives: no pools, empty caches
        return {"vocab": self.vocab, "codec": self.codec, "limit": self.limit}

    def __setstate__(self, st):
        self.__dict__.update(st)
        self.word_ids = {False: {}, True: {}}
        self.pools = {}

    def pool(self, n: int):
        """The text-stage process pool for n workers (started eagerly, once)."""
        pool = self.pools.get(n)
        if pool is None:
            pool = ProcessPoolExecutor(max_workers=n, mp_context=mp.get_context("forkserver"),
                                       initializer=_init_worker, initargs=(self,))
            list(pool.map(_proc_ready, range(n)))
            self.pools[n] = pool
        return pool

    def close(self) -> None:
        for pool in self.pools.values():
            pool.shutdown(wait=False, cancel_futures=True)
        self.pools.clear()

    def __del__(self):
        try:
            self.close()
        except Exception:   # noqa: BLE001 - interpreter teardown
            pass

    def word(self, word: str, pretok: bool) -> tuple:
        toks = [word] if pretok else tokenize_word(word)
        if self.codec is not None:
            toks = bpe_encode(toks, self.codec)
        return tuple(self.vocab.encode(toks))

    def to_ids(self, lines: Sequence[str], pretok: bool) -> "_Chunk":
        """tokenize -> BPE -> vocab ids.  All three stages act word by word
        (textpipe.tokenize splits the cleaned line on whitespace first), so the
        ids of each distinct word are memoised: a Zipfian corpus turns into
        dict lookups after its first few thousand lines."""
        pieces, owner = [], []
        cache = self.word_ids[pretok]
        for li, line in enumerate(lines):
            ids: list = []
            for w in (line.split() if pretok else clean_line(line).split()):
                t = cache.get(w)
                if t is None:
                    t = self.word(w, pretok)
                    if len(cache) < _WORD_CACHE_MAX:
                        cache[w] = t
                ids.extend(t)
            arr = np.asarray(ids, dtype=np.int32)
            for s in range(0, len(arr), self.limit):
                pieces.append(arr[s:s + self.limit])
                owner.append(li)
        return _Chunk(pieces, owner, len(lines))

    def to_text(self, chunk: "_Chunk", outs: list, pretok: bool) -> list:
        per_line = [[] for _ in range(chunk.n_lines)]
        tok = self.vocab.token_of
        for li, ids in zip(chunk.owner, outs):
            per_line[li].extend(tok(int(i)) for i in ids)
        res = []
        for sub in per_line:
            words = bpe_decode(sub) if self.codec is not None else sub
            res.append(" ".join(words) if pretok else detokenize(words))
        return res


class Translator:
    def __init__(self, cfg, weights, vocab: Vocabulary, codec: Optional[BpeCodec] = None,
                 run: RunConfig = RunConfig(), device: int = 0):
        from .engine import Engine
        self.cfg: ModelConfig = config_of(cfg)
        if len(vocab) != self.cfg.vocab_size:
            raise ValueError(f"vocabulary has {len(vocab)} entries, config says "
                             f"{self.cfg.vocab_size}")
        self.vocab = vocab
        self.limit = max(1, min(HARD_SPLIT, self.cfg.max_positions))
        self._text = _TextStage(vocab, codec, self.limit)
        self.run = run
        self.weights = weights
        devs = run.devices if run.devices != (0,) else (device,)
        # one engine (weights + workspace + CUDA graphs) per listed device
        self.engines = [Engine(self.cfg, weights, dtype=run.precision, device=d) for d in devs]
        self.engine = self.engines[0]

    @classmethod
    def from_file(cls, path, run: RunConfig = RunConfig(), bpe_codes=None,
                  device: int = 0) -> "Translator":
        cfg, w, vocab = modelfile.load(path, "int8" if run.precision == "int8" else "f32")
        codec = BpeCodec.load(bpe_codes) if bpe_codes else None
        return cls(cfg, w, vocab, codec=codec, run=run, device=device)

    def with_run(self, **changes) -> "Translator":
        """Same engine (weights stay in HBM), different run flags."""
        t = object.__new__(Translator)
        t.__dict__.update(self.__dict__)
        new = replace(self.run, **changes)
        if new.precision != self.run.precision or new.devices != self.run.devices:
            raise ValueError("precision and devices are fixed at construction "
                             "(weights are uploaded once)")
        t.run = new
        return t

    @property
    def codec(self) -> Optional[BpeCodec]:
        return self._text.codec

    @codec.setter
    def codec(self, value: Optional[BpeCodec]) -> None:   # assignable, like the reference's
        # a fresh stage (caches, pools) for this translator only: with_run copies
        # keep the old codec and its workers
        self._text = _TextStage(self.vocab, value, self.limit)

    def close_pools(self) -> None:
        """Shut down this translator's text-stage workers (recreated on demand)."""
        self._text.close()

    # ---- host stages -------------------------------------------------------
    def _to_ids(self, lines: Sequence[str], pretok: Optional[bool] = None) -> _Chunk:
        pretok = self.run.pretokenized if pretok is None else pretok
        return self._text.to_ids(lines, pretok)

    def _to_text(self, chunk: _Chunk, outs: list, pretok: Optional[bool] = None) -> list:
        pretok = self.run.pretokenized if pretok is None else pretok
        return self._text.to_text(chunk, outs, pretok)

    # ---- GPU stage -----------------------------------------------------------
    def _translate_pieces(self, pieces: list, engine=None) -> list:
        engine = engine or self.engine
        n = len(pieces)
        if n == 0:
            return []
        lengths = np.fromiter((len(p) for p in pieces), dtype=np.int64, count=n)
        offsets = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(lengths, out=offsets[1:])
        ids = np.concatenate(pieces).astype(np.int32) if offsets[-1] else np.zeros(1, np.int32)
        r = self.run
        out_ids, out_len, out_off, _ = engine.translate(
            ids, offsets, sbatch=r.sbatch, wbatch=r.wbatch, ratio=r.max_len_ratio,
            offset=r.max_len_offset, beam=r.beam)
        return [out_ids[o:o + L] for o, L in zip(out_off.tolist(), out_len.tolist())]

    def _groups(self, n_lines: int) -> list:
        """Engine-call groups of whole chunks.  int8 quantizes activations per
        GEMM call over the whole batch (quant8.py:171-195), so its batches are
        kept inside one chunk — the chunk is the unit the reference's worker
        invariance is defined on; the float paths are batch-invariant and
        coalesce chunks into large GPU groups."""
        step = self.run.chunk_lines
        per = 1 if self.run.precision == "int8" else max(1, GPU_GROUP_LINES // step)
        bounds = [(s, min(s + step, n_lines)) for s in range(0, n_lines, step)]
        return [bounds[i:i + per] for i in range(0, len(bounds), per)]

    def translate_lines(self, lines: Sequence[str]) -> list:
        """Groups of chunks go round-robin to the engines (one per device), each
        engine thread translating its groups in order while the text pool
        tokenizes the engine's next group and detokenizes finished ones."""
        lines = list(lines)
        if not lines:
            return []
        groups = self._groups(len(lines))
        n_eng = len(self.engines)
        posted: list = [None] * len(groups)     # per group: futures of detokenized chunks
        pretok = self.run.pretokenized
        procs = self.run.workers > 1
        with ThreadPoolExecutor(max_workers=1 if procs else self.run.workers) as tpool:
            pool = self._text.pool(self.run.workers) if procs else tpool
            pre_fn = _proc_to_ids if procs else self._to_ids
            post_fn = _proc_to_text if procs else self._to_text

            def prep(gi):
                return [pool.submit(pre_fn, lines[s:e], pretok) for s, e in groups[gi]]

            def lane(e):
                mine = list(range(e, len(groups), n_eng))
                pending = prep(mine[0]) if mine else []
                for k, gi in enumerate(mine):
                    try:
                        chunks = [f.result() for f in pending]
                    except Exception as exc:   # noqa: BLE001
                        raise ChunkFailure(gi, exc) from exc
                    if k + 1 < len(mine):
                        pending = prep(mine[k + 1])     # overlaps this group's engine call
                    res = self._translate_pieces([p for c in chunks for p in c.pieces],
                                                 self.engines[e])
                    futs, o = [], 0
                    for c in chunks:
                        futs.append(pool.submit(post_fn, c, res[o:o + len(c.pieces)], pretok))
                        o += len(c.pieces)
                    posted[gi] = futs

            if n_eng == 1:
                lane(0)
            else:
                with ThreadPoolExecutor(max_workers=n_eng) as gpus:
                    for f in [gpus.submit(lane, e) for e in range(n_eng)]:
                        f.result()
            out = [y for futs in posted for f in futs for y in f.result()]
        if len(out) != len(lines):
            raise ChunkFailure(0, ValueError(f"{len(out)} lines out for {len(lines)} in"))
        return out

    # ---- bench / selftest ----------------------------------------------------
    def bench(self, lines: Sequence[str]) -> dict:
        lines = list(lines)
        self.engine.handle  # noqa: B018  (engine built in __init__)
        t0 = time.perf_counter()
        out = self.translate_lines(lines)
        wall = time.perf_counter() - t0
        src_words = sum(len(x.split()) for x in lines)
        tgt_words = sum(len(x.split()) for x in out)
        wall = max(wall, 1e-9)
        return {
            "words_per_second": src_words / wall,
            "wall_seconds": wall,
            "source_words": src_words,
            "source_sentences": len(lines),
            "output_lines": len(out),
            "target_words": tgt_words,
            "target_words_per_second": tgt_words / wall,
            "sentences_per_second": len(lines) / wall,
            "est_peak_bytes": int(max(e.device_bytes() for e in self.engines)),
            "devices": len(self.engines),
            "sbatch": self.run.sbatch,
            "wbatch": self.run.wbatch,
            "workers": self.run.workers,
            "chunk_lines": self.run.chunk_lines,
            "precision": self.run.precision,
            "beam": self.run.beam,
            "device": "cuda",
        }

    def selftest(self) -> list:
        """(name, ok, detail) per case (test_acceptance.py:445-455)."""
        rng = np.random.default_rng(0)
        dirty = bytes(rng.integers(0, 256, size=4096, dtype=np.uint8)).decode(
            "utf-8", errors="replace").replace("\n", " ")
        long_line = ("the quick brown fox jumps over the lazy dog " * 2400)[:100_000]
        cases = [
            ("empty_input", [], lambda o: o == []),
            ("empty_lines", ["", "", ""], lambda o: o == ["", "", ""]),
            ("whitespace_only", ["   \t  "], lambda o: len(o) == 1),
            ("dirty_bytes", [dirty], lambda o: len(o) == 1),
            ("control_chars", ["a\x00b\x07c\x1b[31m d"], lambda o: len(o) == 1),
            ("unknown_words", ["zzz qqq \U0001F600 中文"], lambda o: len(o) == 1),
            ("very_long_line", [long_line, "short"], lambda o: len(o) == 2 and o[0] != ""),
            ("mixed_batch", ["one", "", "two three", "x" * 3000, ""],
             lambda o: len(o) == 5 and o[1] == "" and o[4] == ""),
        ]
        results = []
        for name, lines, ok_fn in cases:
            try:
                out = self.translate_lines(lines)
                ok = bool(ok_fn(out))
                detail = f"lines_in={len(lines)} lines_out={len(out)}"
            except Exception as exc:   # noqa: BLE001 - the battery reports, never raises
                ok, detail = False, f"{type(exc).__name__}: {exc}"
            results.append((name, ok, detail))
        try:
            probe = ["the quick fox", "lazy dog."] * 8
            a = self.translate_lines(probe)
            b = self.with_run(workers=self.run.workers + 3).translate_lines(probe)
            results.append(("worker_invariance", a == b, f"{sum(x == y for x, y in zip(a, b))}"
                                                         f"/{len(a)} identical"))
        except Exception as exc:   # noqa: BLE001
            results.append(("worker_invariance", False, f"{type(exc).__name__}: {exc}"))
        return results


__all__ = ["RunConfig", "Translator", "PRECISIONS", "BOS_ID", "EOS_ID", "PAD_ID"]
