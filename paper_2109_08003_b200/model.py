"""GPU translation model behind the reference's decoding protocol.

``GpuTranslationModel(cfg, weights, dtype="f16")`` is a drop-in for the
reference's ``TranslationModel`` (model.py:370-389): it exposes
``max_positions``, ``encode(tokens, pad_mask)``, ``init_cache(enc)`` and
``step(cache, prev_tokens)``, and its cache supports ``select(rows)``
(model.py:170-181), so the reference's own ``greedy_translate`` /
``beam_translate`` can drive it unchanged.  Every forward FLOP runs in the
CUDA engine (``libfnmt_b200.so``); PyTorch only allocates device buffers.

The fast path — whole batches decoded on the device with a CUDA-graph
captured step, fused vocab-argmax and on-device EOS bookkeeping — is
:meth:`GpuTranslationModel.translate_batch` (used by
:func:`paper_2109_08003_b200.search.greedy_translate`) and the corpus-level
:class:`paper_2109_08003_b200.engine.Engine`.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _capi
from ._capi import check, lib, ptr
from .store import ModelConfig, config_of, iter_named_tensors
from .quant8 import iter_float_tensors, iter_quantized

_TORCH_DT = {_capi.F32: torch.float32, _capi.F16: torch.float16, _capi.BF16: torch.bfloat16,
             _capi.INT8: torch.float32}   # int8 engines keep f32 activations


MAX_DEVICE_BEAM = 8   # fused top-K epilogue width (csrc kTopKMax)


class LengthError(ValueError):
    """Input exceeds the model's position budget (model.py:41-42)."""


def _arch_struct(cfg: ModelConfig) -> _capi.fnmt_arch:
    return _capi.fnmt_arch(cfg.n_enc_layers, cfg.n_dec_layers, cfg.d_model, cfg.n_heads_enc,
                           cfg.n_heads_dec, cfg.ffn_dim_enc, cfg.ffn_dim_dec, cfg.vocab_size,
                           cfg.max_positions, int(cfg.norm_variant == "l1"),
                           int(cfg.shared_embeddings))


class EngineHandle:
    """Owns one ``fnmt_engine`` (device weights + workspace) on one GPU."""

    def __init__(self, cfg, weights, dtype: str = "f16", device: int = 0):
        if not torch.cuda.is_available():
            raise RuntimeError("the B200 engine needs a CUDA device; there is no CPU fallback")
        self.cfg = config_of(cfg)
        self.dtype = _capi.DTYPES[dtype]
        self.device = device
        h = C.c_void_p()
        arch = _arch_struct(self.cfg)
        check(lib.fnmt_engine_create(C.byref(arch), device, self.dtype, C.byref(h)),
              "fnmt_engine_create")
        self.h = h
        if self.dtype == _capi.INT8:
            self._upload_int8(weights)
        else:
            for name, arr in iter_named_tensors(self.cfg, weights):
                arr = np.ascontiguousarray(arr, dtype=np.float32)
                check(lib.fnmt_engine_set_tensor(self.h, name.encode(), arr.ctypes.data,
                                                 arr.size), f"set_tensor({name})")
        check(lib.fnmt_engine_finalize(self.h), "finalize")

    def _upload_int8(self, weights):
        """int8 precision (store.py:29-36): every GEMM weight (and the output
        projection, [d, vocab]) goes up as s8 + per-column scale / zeropoint;
        f32 weights are quantized here, once, like the reference's
        quantize-at-load (store.py:490-524)."""
        for name, arr in iter_float_tensors(self.cfg, weights):
            arr = np.ascontiguousarray(arr, dtype=np.float32)
            check(lib.fnmt_engine_set_tensor(self.h, name.encode(), arr.ctypes.data, arr.size),
                  f"set_tensor({name})")
        for name, qm in iter_quantized(self.cfg, weights):
            q = np.ascontiguousarray(qm.q, dtype=np.int8)
            sc = np.ascontiguousarray(qm.col_scale, dtype=np.float32)
            zp = np.ascontiguousarray(qm.col_zeropoint, dtype=np.float32)
            check(lib.fnmt_engine_set_qtensor(self.h, name.encode(), q.ctypes.data,
                                              sc.ctypes.data, zp.ctypes.data, q.shape[0],
                                              q.shape[1]), f"set_qtensor({name})")

    @property
    def torch_dtype(self):
        return _TORCH_DT[self.dtype]

    def device_bytes(self) -> int:
        return int(lib.fnmt_engine_device_bytes(self.h))

    def close(self):
        if getattr(self, "h", None):
            lib.fnmt_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class GpuEncoderOutput:
    """Encoder output; ``states``/``pad_mask`` behave like the reference's
    EncoderOutput (model.py:148-151).  ``states`` is copied to the host on
    first access."""

    pad_mask: np.ndarray                 # bool [b, s]
    tokens: np.ndarray                   # int64 [b, s] (kept for the fused decode path)
    states_dev: torch.Tensor             # f32 [b, s, d] on the GPU
    states_act: torch.Tensor             # compute dtype [b*s, d] on the GPU
    _host: Optional[np.ndarray] = field(default=None, repr=False)

    @property
    def states(self) -> np.ndarray:
        if self._host is None:
            self._host = self.states_dev.cpu().numpy()
        return self._host

    def row(self, r: int) -> "GpuEncoderOutput":
        s = self.pad_mask.shape[1]
        return GpuEncoderOutput(pad_mask=self.pad_mask[r:r + 1], tokens=self.tokens[r:r + 1],
                                states_dev=self.states_dev[r:r + 1],
                                states_act=self.states_act[r * s:(r + 1) * s])


class GpuDecodeCache:
    """Incremental decoder state on the GPU (model.py:154-181).

    self K/V: per layer [batch, cap, d] in the compute dtype (capacity grows by
    doubling); cross K/V: per layer [batch * src_len, 2d]; row r attends to
    cross rows [k_start[r], k_start[r] + k_len[r]).
    """

    def __init__(self, model, batch, src_len, cross_kv, k_len, cap=None):
        self.model = model
        self.batch = batch
        self.src_len = src_len
        self.cross_kv = cross_kv
        self.k_len = k_len                     # int32 [batch] on GPU
        self.k_start = torch.arange(batch, dtype=torch.int32, device=k_len.device) * src_len
        self.step = 0
        cfg = model.cfg
        self.cap = cap or min(cfg.max_positions, 64)
        self.self_k = [torch.empty((batch, self.cap, cfg.d_model), dtype=model.engine.torch_dtype,
                                   device=k_len.device) for _ in range(cfg.n_dec_layers)]
        self.self_v = [torch.empty_like(t) for t in self.self_k]

    def _grow(self):
        new_cap = min(self.model.cfg.max_positions, self.cap * 2)
        for lst in (self.self_k, self.self_v):
            for i, old in enumerate(lst):
                t = torch.empty((self.batch, new_cap, old.shape[2]), dtype=old.dtype,
                                device=old.device)
                t[:, :self.cap].copy_(old)
                lst[i] = t
        self.cap = new_cap

    def select(self, rows) -> "GpuDecodeCache":
        """New cache holding the given rows (with repetition), for beam search."""
        idx = torch.as_tensor(np.asarray(rows, dtype=np.int32), device=self.k_len.device)
        n = int(idx.numel())
        out = GpuDecodeCache.__new__(GpuDecodeCache)
        out.model, out.batch, out.src_len, out.step, out.cap = (
            self.model, n, self.src_len, self.step, self.cap)
        stream = torch.cuda.current_stream().cuda_stream

        def gather(src, row_elems):
            dst = torch.empty((n,) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
            if n:
                es = src.element_size()
                check(lib.fnmt_gather_rows(ptr(src), ptr(dst), ptr(idx), n, row_elems * es,
                                           row_elems * es, row_elems * es, stream), "select")
            return dst

        d = self.model.cfg.d_model
        out.self_k = [gather(t, self.cap * d) for t in self.self_k]
        out.self_v = [gather(t, self.cap * d) for t in self.self_v]
        out.cross_kv = [gather(t.view(self.batch, -1), self.src_len * 2 * d).view(-1, 2 * d)
                        for t in self.cross_kv]
        out.k_len = gather(self.k_len.view(-1, 1), 1).view(-1)
        out.k_start = torch.arange(n, dtype=torch.int32, device=idx.device) * self.src_len
        torch.cuda.current_stream().synchronize()
        return out


class GpuTranslationModel:
    """Config + device weights behind encode / init_cache / step."""

    def __init__(self, cfg, weights, dtype: str = "f16", device: int = 0):
        self.cfg = config_of(cfg)
        self.engine = EngineHandle(self.cfg, weights, dtype=dtype, device=device)
        self.device = torch.device("cuda", device)

    @property
    def max_positions(self) -> int:
        return self.cfg.max_positions

    def _check_tokens(self, tokens):
        tokens = np.asarray(tokens)
        if tokens.size and (tokens.min() < 0 or tokens.max() >= self.cfg.vocab_size):
            raise ValueError("token id out of range")
        return tokens

    # -- protocol ------------------------------------------------------------

    def encode(self, tokens, pad_mask) -> GpuEncoderOutput:
        tokens = self._check_tokens(tokens)
        pad_mask = np.asarray(pad_mask, dtype=bool)
        b, s = tokens.shape
        if pad_mask.shape != (b, s):
            raise ValueError(f"pad_mask shape {pad_mask.shape} != tokens shape {(b, s)}")
        lens = pad_mask.sum(axis=1)
        if not np.array_equal(pad_mask, np.arange(s)[None, :] < lens[:, None]):
            # the packed-varlen encoder reads row r's keys as its first len_r
            # positions; a left-padded or gapped mask would be silently wrong
            raise ValueError("the GPU engine expects right-padded sources (pad_mask must be "
                             "True on a prefix of each row)")
        if s > self.cfg.max_positions:
            raise LengthError(f"source length {s} exceeds max_positions {self.cfg.max_positions}")
        d = self.cfg.d_model
        tok = torch.as_tensor(tokens.astype(np.int32).reshape(-1), device=self.device)
        lens = torch.as_tensor(pad_mask.sum(axis=1).astype(np.int32), device=self.device)
        states = torch.empty((b, s, d), dtype=torch.float32, device=self.device)
        act = torch.empty((b * s, d), dtype=self.engine.torch_dtype, device=self.device)
        torch.cuda.synchronize(self.device)
        if b * s:
            check(lib.fnmt_engine_encode_padded(self.engine.h, ptr(tok), ptr(lens), b, s,
                                                ptr(states), ptr(act)), "encode")
        return GpuEncoderOutput(pad_mask=pad_mask, tokens=tokens, states_dev=states, states_act=act)

    def init_cache(self, enc: GpuEncoderOutput) -> GpuDecodeCache:
        b, s = enc.pad_mask.shape
        d = self.cfg.d_model
        ckv = []
        for layer in range(self.cfg.n_dec_layers):
            out = torch.empty((b * s, 2 * d), dtype=self.engine.torch_dtype, device=self.device)
            if b * s:
                check(lib.fnmt_engine_cross_kv(self.engine.h, ptr(enc.states_act), b * s, layer,
                                               ptr(out)), "cross_kv")
            ckv.append(out)
        k_len = torch.as_tensor(enc.pad_mask.sum(axis=1).astype(np.int32), device=self.device)
        return GpuDecodeCache(self, b, s, ckv, k_len)

    def step(self, cache: GpuDecodeCache, prev_tokens) -> np.ndarray:
        prev_tokens = self._check_tokens(prev_tokens)
        if prev_tokens.shape != (cache.batch,):
            raise ValueError(f"prev_tokens must be [batch={cache.batch}], got {prev_tokens.shape}")
        t = cache.step
        if t >= self.cfg.max_positions:
            raise LengthError(f"decode position {t} exceeds max_positions {self.cfg.max_positions}")
        while t >= cache.cap:
            cache._grow()
        logits = torch.empty((cache.batch, self.cfg.vocab_size), dtype=torch.float32,
                             device=self.device)
        if cache.batch:
            prev = torch.as_tensor(prev_tokens.astype(np.int32), device=self.device)
            L = self.cfg.n_dec_layers
            kk = (C.c_void_p * L)(*[ptr(x) for x in cache.self_k])
            vv = (C.c_void_p * L)(*[ptr(x) for x in cache.self_v])
            cc = (C.c_void_p * L)(*[ptr(x) for x in cache.cross_kv])
            torch.cuda.synchronize(self.device)
            check(lib.fnmt_engine_decode_step(self.engine.h, ptr(prev), t, cache.batch, cache.cap,
                                              kk, vv, cc, ptr(cache.k_start), ptr(cache.k_len),
                                              cache.src_len, cache.src_len, ptr(logits)),
                  "decode_step")
        cache.step = t + 1
        self._last_logits = logits
        return logits.cpu().numpy()

    def last_step_argmax(self) -> np.ndarray:
        """Device argmax (lowest id on ties) of the logits of the last step()."""
        lg = self._last_logits
        out = torch.empty(lg.shape[0], dtype=torch.int32, device=self.device)
        if lg.shape[0]:
            check(lib.fnmt_argmax_rows(ptr(lg), lg.shape[1], lg.shape[0], lg.shape[1], ptr(out),
                                       torch.cuda.current_stream().cuda_stream), "argmax")
        return out.cpu().numpy()

    def beam_batch(self, enc: GpuEncoderOutput, cfg) -> list[list[int]]:
        """Beam search (search.py:105-147).  Batched on the device: fused
        vocab top-K epilogue, per-sentence selection kernel, ancestor-table
        KV reuse (beam sizes up to MAX_DEVICE_BEAM).  Larger beams, and rows
        whose source is entirely masked (the reference's all-masked attention
        semantics), run the reference's per-sentence search over step()."""
        from .search import _beam_sentence, _device_rows
        rows = _device_rows(self, enc)
        if rows is not None and cfg.beam_size <= MAX_DEVICE_BEAM:
            return self.translate_batch(rows, search=cfg)
        lens = enc.pad_mask.sum(axis=1)
        return [_beam_sentence(self, self.init_cache(enc.row(r)), int(lens[r]), cfg)
                for r in range(enc.pad_mask.shape[0])]

    # -- fused device-side decode ---------------------------------------------

    def translate_batch(self, rows, search=None) -> list[list[int]]:
        """Greedy-translate a list of id sequences in one device-side batch."""
        from .engine import translate_ids
        return translate_ids(self.engine, rows, search=search, sbatch=max(len(rows), 1),
                             wbatch=1 << 30)
