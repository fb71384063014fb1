"""FNMT model files: ``save`` / ``load`` / ``describe`` (store.py:1-26,
:255-536) — the reference's on-disk format, so a model file written by the
reference loads here unchanged and vice versa.

Layout (little-endian; store.py:3-24):

    "FNMT" | u32 version=1
    config   9 x u32 (enc, dec, d, heads_enc, heads_dec, ffn_enc, ffn_dec,
             vocab, max_positions) + u8 norm (0 l2, 1 l1) + u8 shared
    vocab    u32 count, per token u16 byte length + UTF-8
    dir      u32 count, per tensor u16 len + name, u8 dtype (0 f32, 1 qint8),
             u8 ndim, ndim x u32, u64 absolute offset, u64 byte length
    payload  f32 raw row-major | qint8: f32 scale[cols], f32 zp[cols], s8 q[rows*cols]

With shared embeddings ``tgt_embed`` and ``out_proj`` alias ``src_embed``'s
byte range; an int8 file then quantizes the shared projection at load.

B200 notes: loading is host work done once; the GEMM weights then go to HBM
in the engine's layout (``W^T`` K-major, fused QKV) via
:class:`~paper_2109_08003_b200.model.EngineHandle`.  At ``precision="int8"``
the weights stay as :class:`~paper_2109_08003_b200.quant8.QuantizedMatrix`
and are uploaded as s8 + per-column scale / zeropoint for the tcgen05
``kind::i8`` GEMM; at the float precisions an int8 file is dequantized
(lossy, as the reference documents, store.py:512-516).
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass

import numpy as np

from .quant8 import QuantizedMatrix, dequantize_weights, quantize_weights
from .store import (NORM_L1, NORM_L2, AttentionBlock, DecoderLayer, EncoderLayer, FeedForward,
                    ModelConfig, NormParams, Projection, Weights, config_of, sinusoid_positions,
                    tensor_manifest)
from .textpipe import SPECIAL_TOKENS, Vocabulary

MAGIC = b"FNMT"
VERSION = 1
DTYPE_F32, DTYPE_QINT8 = 0, 1
PRECISION_F32, PRECISION_INT8 = "f32", "int8"
PRECISIONS = (PRECISION_F32, PRECISION_INT8)
_CFG = struct.Struct("<9I2B")


class ModelFormatError(ValueError):
    """Not a valid model file of a supported version (store.py:63)."""


@dataclass(frozen=True)
class DirEntry:
    name: str
    dtype: int
    shape: tuple
    offset: int
    nbytes: int


# ----------------------------------------------------------------------------
# write

def _float_of(proj_weight) -> np.ndarray:
    if isinstance(proj_weight, QuantizedMatrix):
        return dequantize_weights(proj_weight)
    return np.asarray(proj_weight, dtype=np.float32)


def _quant_of(proj_weight) -> QuantizedMatrix:
    if isinstance(proj_weight, QuantizedMatrix):
        return proj_weight
    return quantize_weights(np.asarray(proj_weight, dtype=np.float32))


def _q_blob(qm: QuantizedMatrix) -> bytes:
    return (np.asarray(qm.col_scale, "<f4").tobytes() + np.asarray(qm.col_zeropoint, "<f4").tobytes()
            + np.ascontiguousarray(qm.q, dtype=np.int8).tobytes())


def _named_sources(cfg: ModelConfig, w: Weights) -> dict:
    """manifest name -> float array or projection weight (store.py:132-152)."""
    src = {"src_embed": w.src_embed, "tgt_embed": w.tgt_embed, "out_proj": w.out_proj.weight,
           "out_bias": w.out_proj.bias}

    def attn(p, blk):
        for part in "qkvo":
            pr = getattr(blk, part)
            src[f"{p}.{part}_w"], src[f"{p}.{part}_b"] = pr.weight, pr.bias

    def norm(p, n):
        src[f"{p}.gain"], src[f"{p}.bias"] = n.gain, n.bias

    def ffn(p, f):
        src[f"{p}.w1"], src[f"{p}.b1"] = f.w1.weight, f.w1.bias
        src[f"{p}.w2"], src[f"{p}.b2"] = f.w2.weight, f.w2.bias

    for i, L in enumerate(w.enc_layers):
        attn(f"enc.{i}.attn", L.attn)
        norm(f"enc.{i}.norm1", L.norm1)
        ffn(f"enc.{i}.ffn", L.ffn)
        norm(f"enc.{i}.norm2", L.norm2)
    for i, L in enumerate(w.dec_layers):
        attn(f"dec.{i}.self", L.self_attn)
        norm(f"dec.{i}.norm1", L.norm1)
        attn(f"dec.{i}.cross", L.cross_attn)
        norm(f"dec.{i}.norm2", L.norm2)
        if L.ffn is not None:
            ffn(f"dec.{i}.ffn", L.ffn)
            norm(f"dec.{i}.norm3", L.norm3)
    return src


def save(weights: Weights, cfg, path, precision: str = PRECISION_F32,
         vocab: Vocabulary | None = None) -> None:
    """Deterministic writer (store.py:255-335); int8 pre-quantizes every GEMM
    weight (and an unshared output projection)."""
    cfg = config_of(cfg)
    if precision not in PRECISIONS:
        raise ValueError(f"unknown precision {precision!r}")
    vocab = vocab if vocab is not None else Vocabulary()
    if len(vocab) != cfg.vocab_size:
        raise ValueError(f"vocabulary has {len(vocab)} entries, config says {cfg.vocab_size}")
    src = _named_sources(cfg, weights)
    int8 = precision == PRECISION_INT8
    # (name, dtype, shape, blob or None, alias or None)
    items = []
    for name, kind, shape in tensor_manifest(cfg):
        if cfg.shared_embeddings and name in ("tgt_embed", "out_proj"):
            items.append((name, DTYPE_F32, shape, None, "src_embed"))
        elif kind in ("gemm", "out_proj") and int8:
            qm = _quant_of(src[name])             # out_proj: [d, vocab] orientation
            items.append((name, DTYPE_QINT8, (qm.rows, qm.cols), _q_blob(qm), None))
        elif kind == "out_proj":
            arr = np.ascontiguousarray(_float_of(src[name]).T)
            items.append((name, DTYPE_F32, shape, arr.astype("<f4").tobytes(), None))
        elif kind == "gemm":
            items.append((name, DTYPE_F32, shape, _float_of(src[name]).astype("<f4").tobytes(), None))
        else:
            items.append((name, DTYPE_F32, shape,
                          np.asarray(src[name], np.float32).astype("<f4").tobytes(), None))

    head = bytearray(MAGIC + struct.pack("<I", VERSION))
    head += _CFG.pack(cfg.n_enc_layers, cfg.n_dec_layers, cfg.d_model, cfg.n_heads_enc,
                      cfg.n_heads_dec, cfg.ffn_dim_enc, cfg.ffn_dim_dec, cfg.vocab_size,
                      cfg.max_positions, int(cfg.norm_variant == NORM_L1),
                      int(bool(cfg.shared_embeddings)))
    head += struct.pack("<I", len(vocab))
    for tok in vocab.all_tokens():
        b = tok.encode("utf-8")
        head += struct.pack("<H", len(b)) + b
    dir_size = 4 + sum(2 + len(n.encode("utf-8")) + 2 + 4 * len(s) + 16 for n, _, s, _, _ in items)
    cursor = len(head) + dir_size
    spans: dict[str, tuple[int, int]] = {}
    directory = bytearray(struct.pack("<I", len(items)))
    blobs = []
    for name, dt, shape, blob, alias in items:
        if alias is None:
            spans[name] = (cursor, len(blob))
            cursor += len(blob)
            blobs.append(blob)
        else:
            spans[name] = spans[alias]
        nb = name.encode("utf-8")
        directory += struct.pack("<H", len(nb)) + nb + struct.pack("<2B", dt, len(shape))
        directory += struct.pack(f"<{len(shape)}I", *shape) + struct.pack("<2Q", *spans[name])
    try:
        with open(path, "wb") as f:
            f.write(bytes(head))
            f.write(bytes(directory))
            for b in blobs:
                f.write(b)
    except OSError as exc:
        raise OSError(f"cannot write model to {path}: {exc}") from exc


# ----------------------------------------------------------------------------
# read

class _Reader:
    def __init__(self, buf: bytes, path):
        self.buf, self.pos, self.path = buf, 0, path

    def take(self, fmt: str):
        try:
            vals = struct.unpack_from(fmt, self.buf, self.pos)
        except struct.error as exc:
            raise ModelFormatError(f"{self.path}: truncated header") from exc
        self.pos += struct.calcsize(fmt)
        return vals

    def raw(self, n: int) -> bytes:
        if self.pos + n > len(self.buf):
            raise ModelFormatError(f"{self.path}: truncated header")
        b = self.buf[self.pos:self.pos + n]
        self.pos += n
        return b


def _parse(buf: bytes, path):
    if len(buf) < 8 or buf[:4] != MAGIC:
        raise ModelFormatError(f"{path}: bad magic")
    r = _Reader(buf, path)
    r.pos = 4
    (version,) = r.take("<I")
    if version != VERSION:
        raise ModelFormatError(f"{path}: unsupported version {version}")
    f = r.take(_CFG.format)
    cfg = ModelConfig(*f[:9], norm_variant=NORM_L1 if f[9] else NORM_L2,
                      shared_embeddings=bool(f[10]))
    (nv,) = r.take("<I")
    toks = []
    for _ in range(nv):
        (ln,) = r.take("<H")
        toks.append(r.raw(ln).decode("utf-8"))
    if toks[:len(SPECIAL_TOKENS)] != list(SPECIAL_TOKENS):
        raise ModelFormatError(f"{path}: vocabulary lacks the special tokens")
    vocab = Vocabulary(toks[len(SPECIAL_TOKENS):])
    if len(vocab) != cfg.vocab_size:
        raise ModelFormatError(f"{path}: vocabulary size {len(vocab)} != config vocab "
                               f"{cfg.vocab_size}")
    (nt,) = r.take("<I")
    entries = []
    for _ in range(nt):
        (ln,) = r.take("<H")
        name = r.raw(ln).decode("utf-8")
        dt, nd = r.take("<2B")
        shape = tuple(r.take(f"<{nd}I"))
        off, nb = r.take("<2Q")
        entries.append(DirEntry(name, dt, shape, off, nb))
    return cfg, vocab, entries


def _check(cfg: ModelConfig, entries, size: int, path) -> dict:
    by = {}
    for e in entries:
        if e.name in by:
            raise ModelFormatError(f"{path}: duplicate tensor {e.name}")
        by[e.name] = e
    want = {n for n, _, _ in tensor_manifest(cfg)}
    if want - by.keys():
        raise ModelFormatError(f"{path}: missing tensor {sorted(want - by.keys())[0]}")
    if by.keys() - want:
        raise ModelFormatError(f"{path}: unexpected tensor {sorted(by.keys() - want)[0]}")
    for e in entries:
        if e.dtype == DTYPE_F32:
            need = 4 * math.prod(e.shape)
        elif e.dtype == DTYPE_QINT8 and len(e.shape) == 2:
            need = 8 * e.shape[1] + e.shape[0] * e.shape[1]
        else:
            raise ModelFormatError(f"{path}: tensor {e.name} has unknown dtype {e.dtype}")
        if e.nbytes != need:
            raise ModelFormatError(f"{path}: tensor {e.name} has inconsistent byte length")
        if e.offset + e.nbytes > size:
            raise ModelFormatError(f"{path}: tensor {e.name} is truncated")
    prev = None
    for cur in sorted((e.offset, e.nbytes, e.name) for e in entries):
        if prev is not None and not (prev[:2] == cur[:2]) and cur[0] < prev[0] + prev[1]:
            raise ModelFormatError(f"{path}: tensors {prev[2]} and {cur[2]} overlap")
        prev = cur
    if cfg.shared_embeddings:
        s = by["src_embed"]
        for alias in ("tgt_embed", "out_proj"):
            if (by[alias].offset, by[alias].nbytes) != (s.offset, s.nbytes):
                raise ModelFormatError(
                    f"{path}: {alias} must alias src_embed in a shared-embeddings model")
    if by["src_embed"].dtype != DTYPE_F32:
        raise ModelFormatError(f"{path}: embeddings must be stored as f32")
    return by


def _array(buf: bytes, e: DirEntry):
    if e.dtype == DTYPE_F32:
        return np.frombuffer(buf, "<f4", math.prod(e.shape), e.offset).reshape(e.shape)
    k, n = e.shape
    scale = np.frombuffer(buf, "<f4", n, e.offset).astype(np.float32)
    zp = np.frombuffer(buf, "<f4", n, e.offset + 4 * n).astype(np.float32)
    q = np.frombuffer(buf, np.int8, k * n, e.offset + 8 * n).reshape(k, n)
    return QuantizedMatrix(k, n, q, scale, zp)


def _projection(w, bias, precision: str) -> Projection:
    bias = np.asarray(bias, np.float32)
    if precision == PRECISION_INT8:
        return Projection(w if isinstance(w, QuantizedMatrix) else quantize_weights(w), bias)
    return Projection(_float_of(w), bias)


def _assemble(cfg: ModelConfig, a: dict, precision: str) -> Weights:
    out_w = a["out_proj"]
    if not isinstance(out_w, QuantizedMatrix):
        out_w = np.asarray(out_w, np.float32).T          # stored [vocab, d]
    P = lambda w, b: _projection(a[w], a[b], precision)   # noqa: E731
    N = lambda p: NormParams(np.asarray(a[p + ".gain"], np.float32),   # noqa: E731
                             np.asarray(a[p + ".bias"], np.float32))
    att = lambda p: AttentionBlock(*(P(f"{p}.{x}_w", f"{p}.{x}_b") for x in "qkvo"))  # noqa: E731
    enc = [EncoderLayer(att(f"enc.{i}.attn"), N(f"enc.{i}.norm1"),
                        FeedForward(P(f"enc.{i}.ffn.w1", f"enc.{i}.ffn.b1"),
                                    P(f"enc.{i}.ffn.w2", f"enc.{i}.ffn.b2")),
                        N(f"enc.{i}.norm2")) for i in range(cfg.n_enc_layers)]
    has = cfg.ffn_dim_dec > 0
    dec = [DecoderLayer(att(f"dec.{i}.self"), N(f"dec.{i}.norm1"), att(f"dec.{i}.cross"),
                        N(f"dec.{i}.norm2"),
                        FeedForward(P(f"dec.{i}.ffn.w1", f"dec.{i}.ffn.b1"),
                                    P(f"dec.{i}.ffn.w2", f"dec.{i}.ffn.b2")) if has else None,
                        N(f"dec.{i}.norm3") if has else None) for i in range(cfg.n_dec_layers)]
    return Weights(src_embed=np.asarray(a["src_embed"], np.float32),
                   tgt_embed=np.asarray(a["tgt_embed"], np.float32),
                   out_proj=_projection(out_w, a["out_bias"], precision),
                   enc_layers=enc, dec_layers=dec,
                   positions=sinusoid_positions(cfg.max_positions, cfg.d_model))


def load(path, precision: str = PRECISION_F32):
    """-> (ModelConfig, Weights, Vocabulary) (store.py:490-524)."""
    if precision not in PRECISIONS:
        raise ValueError(f"unknown precision {precision!r}")
    try:
        with open(path, "rb") as f:
            buf = f.read()
    except OSError as exc:
        raise OSError(f"cannot read model from {path}: {exc}") from exc
    cfg, vocab, entries = _parse(buf, path)
    by = _check(cfg, entries, len(buf), path)
    arrays = {name: _array(buf, e) for name, e in by.items()}
    return cfg, _assemble(cfg, arrays, precision), vocab


def describe(path) -> str:
    with open(path, "rb") as f:
        buf = f.read()
    cfg, vocab, entries = _parse(buf, path)
    out = [f"version={VERSION} file_bytes={len(buf)}",
           f"config: enc_layers={cfg.n_enc_layers} dec_layers={cfg.n_dec_layers}"
           f" d_model={cfg.d_model} heads={cfg.n_heads_enc}/{cfg.n_heads_dec}"
           f" ffn={cfg.ffn_dim_enc}/{cfg.ffn_dim_dec} vocab={cfg.vocab_size}"
           f" max_positions={cfg.max_positions} norm={cfg.norm_variant}"
           f" shared_embeddings={cfg.shared_embeddings}",
           f"vocabulary: {len(vocab)} tokens",
           f"tensors: {len(entries)}"]
    for e in entries:
        out.append(f"  {e.name}  dtype={'f32' if e.dtype == DTYPE_F32 else 'qint8'} "
                   f"shape={'x'.join(map(str, e.shape))} offset={e.offset} bytes={e.nbytes}")
    return "\n".join(out)
