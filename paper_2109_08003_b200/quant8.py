"""Per-column int8 weight quantization (host side, load time).

Same scheme as the reference ``fastnmt.quant8`` (quant8.py:1-278, the
paper's Eqs. 3-6): column j of a ``[k, n]`` weight maps to signed 8 bits with
``scale_j = 14 sigma_j / 255`` (stored f32) and zeropoint
``-0.5 - mean_j / scale_j`` (stored f32), rounding half away from zero
(quant8.py:132-168); degenerate columns take scale 1, zeropoint -mean.

Only the *weight* side lives here: weights are quantized once when a model is
loaded at ``precision="int8"`` (or read pre-quantized from an int8 model
file) and uploaded to HBM.  The per-call activation quantization and the
integer GEMM run on the GPU (``csrc/qgemm.cu``): ``fnmt_qgemm`` computes the
same ``dequantize(a) @ dequantize(b)`` identity (quant8.py:246-278) with
u8 x s8 -> s32 tcgen05 MMAs, bit-exact in the integer core.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterator

import numpy as np


def round_half_away(x) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    return np.trunc(x + np.copysign(0.5, x))


@dataclass(frozen=True)
class QuantizedMatrix:
    rows: int
    cols: int
    q: np.ndarray               # int8 [rows, cols]  (k-major rows, like the f32 weight)
    col_scale: np.ndarray       # f32 [cols]
    col_zeropoint: np.ndarray   # f32 [cols]


def quantize_weights(w: np.ndarray) -> QuantizedMatrix:
    w = np.asarray(w, dtype=np.float32)
    if w.ndim != 2 or w.shape[0] < 1:
        raise ValueError(f"quantize_weights expects a [k, n] matrix, got {w.shape}")
    mu = w.mean(axis=0, dtype=np.float64)
    sd = w.std(axis=0, dtype=np.float64)
    scale = (14.0 * sd / 255.0).astype(np.float32)
    bad = ~(np.isfinite(scale) & (scale > 0))
    scale = np.where(bad, np.float32(1.0), scale).astype(np.float32)
    zp = np.where(bad, -mu, -0.5 - mu / scale.astype(np.float64)).astype(np.float32)
    lv = round_half_away(w.astype(np.float64) / scale.astype(np.float64) +
                         zp.astype(np.float64))
    q = np.clip(lv, -128, 127).astype(np.int8)
    return QuantizedMatrix(w.shape[0], w.shape[1], q, scale, zp)


def dequantize_weights(qm: QuantizedMatrix) -> np.ndarray:
    return ((qm.q.astype(np.float64) - qm.col_zeropoint.astype(np.float64)[None, :]) *
            qm.col_scale.astype(np.float64)[None, :]).astype(np.float32)


def as_quantized(weight) -> QuantizedMatrix:
    """A projection weight as a QuantizedMatrix: f32 [k, n] arrays are
    quantized (quantize-at-load), QuantizedMatrix passes through, and the
    reference's PackedMatrix (quant8.py:85-109) is read through its
    ``gemm_operand`` (the exact levels as f32) and column statistics."""
    if isinstance(weight, QuantizedMatrix):
        return weight
    if hasattr(weight, "gemm_operand") and hasattr(weight, "col_scale"):
        q = np.asarray(weight.gemm_operand).astype(np.int8)
        return QuantizedMatrix(q.shape[0], q.shape[1], q,
                               np.asarray(weight.col_scale, np.float32),
                               np.asarray(weight.col_zeropoint, np.float32))
    return quantize_weights(np.asarray(weight, dtype=np.float32))


def iter_quantized(cfg, w) -> Iterator[tuple]:
    """(name, QuantizedMatrix) for every GEMM weight in the reference
    orientation, plus ``out_proj`` as the [d, vocab] projection (store.py:
    268-285: the int8 model quantizes the shared output projection too)."""
    yield "out_proj", as_quantized(w.out_proj.weight)

    def block(prefix, blk):
        for part in "qkvo":
            yield f"{prefix}.{part}_w", as_quantized(getattr(blk, part).weight)

    for i, L in enumerate(w.enc_layers):
        yield from block(f"enc.{i}.attn", L.attn)
        yield f"enc.{i}.ffn.w1", as_quantized(L.ffn.w1.weight)
        yield f"enc.{i}.ffn.w2", as_quantized(L.ffn.w2.weight)
    for i, L in enumerate(w.dec_layers):
        yield from block(f"dec.{i}.self", L.self_attn)
        yield from block(f"dec.{i}.cross", L.cross_attn)
        if L.ffn is not None:
            yield f"dec.{i}.ffn.w1", as_quantized(L.ffn.w1.weight)
            yield f"dec.{i}.ffn.w2", as_quantized(L.ffn.w2.weight)


def iter_float_tensors(cfg, w):
    """The f32 tensors of an int8 model: embeddings, biases, norms, positions."""
    from .store import iter_named_tensors
    return iter_named_tensors(cfg, w, skip_gemm=True)


def device_operands(qm: QuantizedMatrix):
    """Host arrays of ``fnmt_qgemm``'s weight operand: s8 W^T [n, Kp] (K
    zero-padded to 16), scale [n], zeropoint [n], s32 level sums [n]."""
    k, n = qm.q.shape
    kp = (k + 15) // 16 * 16
    wt = np.zeros((n, kp), np.int8)
    wt[:, :k] = np.asarray(qm.q, np.int8).T
    colsum = np.asarray(qm.q, np.int64).sum(axis=0).astype(np.int32)
    return (wt, np.ascontiguousarray(qm.col_scale, np.float32),
            np.ascontiguousarray(qm.col_zeropoint, np.float32), colsum)
