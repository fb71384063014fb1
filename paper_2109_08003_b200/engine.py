"""Corpus-level translation on the B200 engine.

``Engine`` wraps one ``fnmt_engine`` per GPU and exposes the reference's
batch-translate contract at the id level: length-sorted token-budget
batching (batching.py:100-109), greedy decode of every batch
(search.py:58-86) and order restoration (batching.py:112-122) — all inside
one native call.  Two entry points, matching the two halves of the bench:

* :meth:`Engine.translate` — host (numpy / pinned torch) buffers in and out;
  the host<->device copies happen inside the call (the ``e2e`` path);
* :meth:`Engine.translate_device` — inputs and outputs already in HBM.

``RunConfig`` (defined in ``translator.py``) mirrors the reference's run
flags (cli.py:20-45) with the GPU decoding caps of the paper (sbatch 3072 /
wbatch 64000).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _capi
from ._capi import check, lib, ptr
from .store import BOS_ID, EOS_ID, PAD_ID
from .translator import RunConfig  # noqa: F401  (re-export; cli.py:34-45)


def run_struct(sbatch, wbatch, ratio=1.5, offset=5, beam=1, bos=BOS_ID, eos=EOS_ID,
               pad=PAD_ID) -> _capi.fnmt_run:
    return _capi.fnmt_run(int(sbatch), int(wbatch), float(ratio), int(offset), int(beam),
                          int(bos), int(eos), int(pad))


def budgets_of(lengths: np.ndarray, ratio: float, offset: int, max_positions: int) -> np.ndarray:
    lengths = np.ascontiguousarray(lengths, dtype=np.int32)
    out = np.empty_like(lengths)
    check(lib.fnmt_budgets(lengths.ctypes.data, len(lengths), float(ratio), int(offset),
                           int(max_positions), out.ctypes.data), "budgets")
    return out


def native_plan(lengths, sbatch: int, wbatch: int):
    """The native scheduler's batch plan (``fnmt_plan_batches``, host only):
    returns ``(permutation, batches)`` with ``batches`` a list of
    ``(indices, max_len, oversize)`` — the shape of ``batching.plan_batches``
    (batching.py:100-109), so the planner ``fnmt_engine_translate`` runs can be
    checked against the reference's fixtures without a GPU."""
    lengths = np.ascontiguousarray(lengths, dtype=np.int32)
    n = len(lengths)
    perm = np.empty(max(n, 1), np.int32)
    sizes = np.empty(max(n, 1), np.int32)
    mlen = np.empty(max(n, 1), np.int32)
    over = np.empty(max(n, 1), np.uint8)
    k = check(lib.fnmt_plan_batches(lengths.ctypes.data, n, int(sbatch), int(wbatch),
                                    perm.ctypes.data, sizes.ctypes.data, mlen.ctypes.data,
                                    over.ctypes.data), "plan_batches")
    batches, j = [], 0
    for b in range(k):
        batches.append((perm[j:j + sizes[b]].tolist(), int(mlen[b]), bool(over[b])))
        j += int(sizes[b])
    return perm[:n].tolist(), batches


def stats_dict(st: _capi.fnmt_stats) -> dict:
    return {name: getattr(st, name) for name, _ in st._fields_}


class Engine:
    """Native corpus translator on one GPU."""

    def __init__(self, cfg, weights, dtype: str = "f16", device: int = 0):
        from .model import EngineHandle
        self.handle = weights if isinstance(weights, EngineHandle) else EngineHandle(
            cfg, weights, dtype=dtype, device=device)
        self.cfg = self.handle.cfg

    def reserve(self, sbatch=3072, wbatch=64000, ratio=1.5, offset=5):
        r = run_struct(sbatch, wbatch, ratio, offset)
        check(lib.fnmt_engine_reserve(self.handle.h, C.byref(r)), "reserve")

    def plan_outputs(self, lengths, ratio=1.5, offset=5):
        b = budgets_of(lengths, ratio, offset, self.cfg.max_positions)
        off = np.zeros(len(b), dtype=np.int64)
        if len(b):
            np.cumsum(b[:-1], out=off[1:])
        return b, off

    def translate(self, ids: np.ndarray, offsets: np.ndarray, sbatch=3072, wbatch=64000,
                  ratio=1.5, offset=5, out_ids=None, out_len=None, out_off=None, beam=1):
        """Host buffers.  ids int32 (flat), offsets int64 [n+1].  Returns
        (out_ids flat int32 laid out at out_off, out_len int32 [n], out_off, stats).
        beam > 1 runs the batched device beam search (search.py:105-147)."""
        ids = np.ascontiguousarray(ids, dtype=np.int32) if isinstance(ids, np.ndarray) else ids
        offsets = np.ascontiguousarray(offsets, dtype=np.int64) if isinstance(
            offsets, np.ndarray) else offsets
        n = len(offsets) - 1
        lengths = np.diff(np.asarray(offsets)).astype(np.int32)
        b, planned_off = self.plan_outputs(lengths, ratio, offset)
        if out_off is None:
            out_off = planned_off
        else:
            out_off = np.ascontiguousarray(out_off, dtype=np.int64)
            if out_off.shape != (n,) or (n and out_off.min() < 0):
                raise ValueError(f"out_off must be {n} non-negative int64 offsets")
        # the native call writes sentence i's ids at out_ids[out_off[i] : +budget_i]
        total = int((out_off + b).max()) if n else 0
        if out_ids is None:
            out_ids = np.empty(max(total, 1), dtype=np.int32)
        elif len(out_ids) < total:
            raise ValueError(f"out_ids holds {len(out_ids)} ids, the budgets need {total}")
        if out_len is None:
            out_len = np.empty(max(n, 1), dtype=np.int32)
        elif len(out_len) < n:
            raise ValueError(f"out_len holds {len(out_len)} entries, need {n}")
        st = _capi.fnmt_stats()
        r = run_struct(sbatch, wbatch, ratio, offset, beam)
        check(lib.fnmt_engine_translate(self.handle.h, ptr(ids), ptr(offsets), n, C.byref(r),
                                        ptr(out_ids), ptr(out_off), ptr(out_len), C.byref(st)),
              "translate")
        return out_ids, out_len, out_off, st

    def translate_device(self, d_ids: torch.Tensor, d_offsets: torch.Tensor, lengths: np.ndarray,
                         d_out_ids: torch.Tensor, out_off: np.ndarray, d_out_off: torch.Tensor,
                         d_out_len: torch.Tensor, sbatch=3072, wbatch=64000, ratio=1.5, offset=5,
                         beam=1):
        lengths = np.ascontiguousarray(lengths, dtype=np.int32)
        st = _capi.fnmt_stats()
        r = run_struct(sbatch, wbatch, ratio, offset, beam)
        check(lib.fnmt_engine_translate_device(
            self.handle.h, ptr(d_ids), ptr(d_offsets), lengths.ctypes.data, len(lengths),
            C.byref(r), ptr(d_out_ids), out_off.ctypes.data, ptr(d_out_off), ptr(d_out_len),
            C.byref(st)), "translate_device")
        return st

    def device_bytes(self) -> int:
        return self.handle.device_bytes()

    def profile(self, on: bool = True):
        """Bracket every engine launch with CUDA events (decode runs un-captured)."""
        check(lib.fnmt_engine_profile(self.handle.h, int(on)), "profile")

    def profile_read(self) -> dict:
        n = len(_capi.KERNEL_CLASSES)
        ms, cnt = (C.c_double * n)(), (C.c_int64 * n)()
        fl, by = (C.c_double * n)(), (C.c_double * n)()
        check(lib.fnmt_engine_profile_read(self.handle.h, ms, cnt, fl, by), "profile_read")
        return {name: {"ms": ms[i], "launches": cnt[i], "flops": fl[i], "bytes": by[i]}
                for i, name in enumerate(_capi.KERNEL_CLASSES)}


    def profile_log(self) -> dict:
        """Per-launch log of the profiled runs (launch order): numpy arrays
        ``cls`` (index into KERNEL_CLASSES), ``ms``, ``flops``, ``bytes``."""
        n = check(lib.fnmt_engine_profile_log(self.handle.h, None, None, None, None, 0),
                  "profile_log")
        out = {"cls": np.empty(n, np.int32), "ms": np.empty(n, np.float32),
               "flops": np.empty(n, np.float64), "bytes": np.empty(n, np.float64)}
        check(lib.fnmt_engine_profile_log(self.handle.h, out["cls"].ctypes.data,
                                          out["ms"].ctypes.data, out["flops"].ctypes.data,
                                          out["bytes"].ctypes.data, n), "profile_log")
        return out

def translate_ids(handle, rows, search=None, sbatch=3072, wbatch=64000) -> list[list[int]]:
    """Translate a list of id sequences through the native corpus path (greedy,
    or batched beam when search.beam_size > 1)."""
    beam = getattr(search, "beam_size", 1)
    ratio = getattr(search, "max_len_ratio", 1.5)
    offset = getattr(search, "max_len_offset", 5)
    bos = getattr(search, "bos_id", BOS_ID)
    eos = getattr(search, "eos_id", EOS_ID)
    pad = getattr(search, "pad_id", PAD_ID)
    rows = [np.asarray(r, dtype=np.int64) for r in rows]
    n = len(rows)
    if n == 0:
        return []
    lengths = np.array([len(r) for r in rows], dtype=np.int32)
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lengths, out=offsets[1:])
    ids = np.concatenate(rows).astype(np.int32) if offsets[-1] else np.zeros(1, np.int32)
    cfg = handle.cfg
    if ids.size and offsets[-1] and (ids.min() < 0 or ids.max() >= cfg.vocab_size):
        raise ValueError("token id out of range")
    budgets = budgets_of(lengths, ratio, offset, cfg.max_positions)
    out_off = np.zeros(n, dtype=np.int64)
    np.cumsum(budgets[:-1], out=out_off[1:])
    out_ids = np.empty(max(int(budgets.sum()), 1), dtype=np.int32)
    out_len = np.empty(n, dtype=np.int32)
    st = _capi.fnmt_stats()
    r = run_struct(sbatch, min(wbatch, int(lengths.max(initial=1)) * n), ratio, offset, beam, bos,
                   eos, pad)
    check(lib.fnmt_engine_translate(handle.h, ids.ctypes.data, offsets.ctypes.data, n,
                                    C.byref(r), out_ids.ctypes.data, out_off.ctypes.data,
                                    out_len.ctypes.data, C.byref(st)), "translate")
    return [out_ids[o:o + L].tolist() for o, L in zip(out_off, out_len)]
