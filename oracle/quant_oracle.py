"""CPU restatement of the reference's int8 scheme — TEST INFRASTRUCTURE ONLY
(imported by tests/ as the checker; never by the product path).

Follows /root/reference/pkg/src/fastnmt/quant8.py:
  * round half away from zero            quant8.py:112-115
  * quantize_weights (per column, s8)    quant8.py:132-168
  * quantize_activations (per matrix, u8) quant8.py:171-195
  * qgemm (exact integer core, zeropoint cross terms, f64 scale) quant8.py:246-278
Pinned bit-exact against tests/golden/quant8.npz (oracle/make_golden_quant.py,
which ran the reference itself).
"""

from __future__ import annotations

import numpy as np


def rha(x):
    x = np.asarray(x, np.float64)
    return np.trunc(x + np.copysign(0.5, x))


def quantize_weights(w):
    """-> (q s8 [k, n], scale f32 [n], zp f32 [n])"""
    w = np.asarray(w, np.float32)
    mean = w.mean(axis=0, dtype=np.float64)
    std = w.std(axis=0, dtype=np.float64)
    scale = (14.0 * std / 255.0).astype(np.float32)
    bad = ~(np.isfinite(scale) & (scale > 0))
    scale = np.where(bad, np.float32(1.0), scale)
    zp = np.where(bad, -mean, -0.5 - mean / scale.astype(np.float64)).astype(np.float32)
    q = np.clip(rha(w.astype(np.float64) / scale.astype(np.float64) + zp.astype(np.float64)),
                -128, 127).astype(np.int8)
    return q, scale, zp


def quantize_activations(x):
    """-> (q u8 [m, k], scale float, zp float)"""
    x = np.asarray(x, np.float32)
    hi, lo = float(x.max()), float(x.min())
    if hi == lo:
        scale, zp = 1.0, 255.0 - hi
    else:
        scale = (hi - lo) / 255.0
        zp = 255.0 - hi / scale
    q = np.clip(rha(x.astype(np.float64) / scale + zp), 0, 255).astype(np.uint8)
    return q, scale, zp


def qgemm(aq, ascale, azp, wq, wscale, wzp):
    """f32 [m, n] = dequant(a) @ dequant(w), integer core exact."""
    k = aq.shape[1]
    acc = aq.astype(np.int64) @ wq.astype(np.int64)          # exact
    acc = acc.astype(np.float64)
    rows = aq.astype(np.int64).sum(axis=1).astype(np.float64)[:, None]
    cols = wq.astype(np.int64).sum(axis=0).astype(np.float64)[None, :]
    bz = wzp.astype(np.float64)[None, :]
    corr = acc - bz * rows - azp * cols + k * azp * bz
    return ((ascale * wscale.astype(np.float64)[None, :]) * corr).astype(np.float32)


def linear(x, w, bias=None):
    """Projection.apply on a quantized weight (model.py:84-90)."""
    q, s, z = quantize_weights(w)
    aq, asc, azp = quantize_activations(x)
    out = qgemm(aq, asc, azp, q, s, z)
    return out if bias is None else out + np.asarray(bias, np.float32)
