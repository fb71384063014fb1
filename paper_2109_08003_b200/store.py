"""Model configuration and construction (host side).

Mirrors the reference's construction entry points so users can switch
without touching their setup code:

* ``ModelConfig`` — same fields and validation as model.py:45-70;
* ``count_params`` — model.py:347-367;
* ``tensor_manifest`` — store.py:88-115 (names, kinds, logical shapes, and the
  order ``random_model`` draws them in);
* ``random_model(cfg, seed)`` — store.py:539-572: the same PCG64 stream and
  draw order, so the weights are bit-identical to the reference's;
* ``Weights`` and friends — duck-type compatible with the reference's weight
  dataclasses (model.py:93-145): a reference ``Weights`` object can be handed
  to :class:`GpuTranslationModel` unchanged, and vice versa.

This is one-time host work (the reference does it on the CPU too); all
forward/decode compute runs in the CUDA engine.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Iterator, Optional

import numpy as np

NORM_L2, NORM_L1 = "l2", "l1"
PAD_ID, UNK_ID, BOS_ID, EOS_ID = 0, 1, 2, 3          # textpipe.py:43-45


@dataclass(frozen=True)
class ModelConfig:
    n_enc_layers: int
    n_dec_layers: int
    d_model: int
    n_heads_enc: int
    n_heads_dec: int
    ffn_dim_enc: int
    ffn_dim_dec: int
    vocab_size: int
    max_positions: int
    norm_variant: str = NORM_L2
    shared_embeddings: bool = True

    def __post_init__(self):
        must_be_positive = (self.n_enc_layers, self.n_dec_layers, self.d_model, self.n_heads_enc,
                            self.n_heads_dec, self.ffn_dim_enc, self.vocab_size,
                            self.max_positions)
        if min(must_be_positive) < 1:
            raise ValueError("all sizes except ffn_dim_dec must be >= 1")
        if self.ffn_dim_dec < 0:
            raise ValueError("ffn_dim_dec must be >= 0")
        if self.d_model % self.n_heads_enc or self.d_model % self.n_heads_dec:
            raise ValueError("d_model must be divisible by both head counts")
        if self.norm_variant not in (NORM_L2, NORM_L1):
            raise ValueError(f"unknown norm variant {self.norm_variant!r}")


def config_of(cfg) -> ModelConfig:
    """Accept a reference ModelConfig (or anything with the same fields)."""
    if isinstance(cfg, ModelConfig):
        return cfg
    return ModelConfig(**{f: getattr(cfg, f) for f in ModelConfig.__dataclass_fields__})


def count_params(cfg: ModelConfig) -> int:
    d, f_e, f_d = cfg.d_model, cfg.ffn_dim_enc, cfg.ffn_dim_dec
    dense = lambda i, o: i * o + o
    per_enc = 4 * dense(d, d) + dense(d, f_e) + dense(f_e, d) + 2 * (2 * d)
    per_dec = 8 * dense(d, d) + 2 * (2 * d)
    if f_d > 0:
        per_dec += dense(d, f_d) + dense(f_d, d) + 2 * d
    tables = cfg.vocab_size * d * (1 if cfg.shared_embeddings else 3)
    return tables + cfg.vocab_size + cfg.n_enc_layers * per_enc + cfg.n_dec_layers * per_dec


# --- weight containers (attribute-compatible with model.py:73-145) ---------

@dataclass
class Projection:
    weight: np.ndarray      # [k, n] float32 (x @ weight)
    bias: np.ndarray        # [n]


@dataclass
class NormParams:
    gain: np.ndarray
    bias: np.ndarray


@dataclass
class AttentionBlock:
    q: Projection
    k: Projection
    v: Projection
    o: Projection


@dataclass
class FeedForward:
    w1: Projection
    w2: Projection


@dataclass
class EncoderLayer:
    attn: AttentionBlock
    norm1: NormParams
    ffn: FeedForward
    norm2: NormParams


@dataclass
class DecoderLayer:
    self_attn: AttentionBlock
    norm1: NormParams
    cross_attn: AttentionBlock
    norm2: NormParams
    ffn: Optional[FeedForward] = None
    norm3: Optional[NormParams] = None


@dataclass
class Weights:
    src_embed: np.ndarray
    tgt_embed: np.ndarray
    out_proj: Projection     # weight is the [d, vocab] transposed view of the table
    enc_layers: list = field(default_factory=list)
    dec_layers: list = field(default_factory=list)
    positions: Optional[np.ndarray] = None


def sinusoid_positions(max_positions: int, d_model: int) -> np.ndarray:
    """Interleaved table (sin at even columns, cos at odd), model.py:184-190."""
    col = np.arange(d_model, dtype=np.float64)
    denom = np.power(10000.0, (2.0 * np.floor(col / 2.0)) / d_model)
    angle = np.arange(max_positions, dtype=np.float64)[:, None] / denom[None, :]
    even = (np.arange(d_model) % 2 == 0)[None, :]
    return np.where(even, np.sin(angle), np.cos(angle)).astype(np.float32)


def tensor_manifest(cfg: ModelConfig) -> list[tuple[str, str, tuple[int, ...]]]:
    d, v = cfg.d_model, cfg.vocab_size
    out: list[tuple[str, str, tuple[int, ...]]] = [
        ("src_embed", "embed", (v, d)), ("tgt_embed", "embed", (v, d)),
        ("out_proj", "out_proj", (v, d)), ("out_bias", "plain", (v,))]

    def block(prefix):
        for part in ("q", "k", "v", "o"):
            out.extend([(f"{prefix}.{part}_w", "gemm", (d, d)), (f"{prefix}.{part}_b", "plain", (d,))])

    def norm(prefix):
        out.extend([(f"{prefix}.gain", "plain", (d,)), (f"{prefix}.bias", "plain", (d,))])

    def ffn(prefix, width):
        out.extend([(f"{prefix}.w1", "gemm", (d, width)), (f"{prefix}.b1", "plain", (width,)),
                    (f"{prefix}.w2", "gemm", (width, d)), (f"{prefix}.b2", "plain", (d,))])

    for i in range(cfg.n_enc_layers):
        block(f"enc.{i}.attn"); norm(f"enc.{i}.norm1")
        ffn(f"enc.{i}.ffn", cfg.ffn_dim_enc); norm(f"enc.{i}.norm2")
    for i in range(cfg.n_dec_layers):
        block(f"dec.{i}.self"); norm(f"dec.{i}.norm1")
        block(f"dec.{i}.cross"); norm(f"dec.{i}.norm2")
        if cfg.ffn_dim_dec > 0:
            ffn(f"dec.{i}.ffn", cfg.ffn_dim_dec); norm(f"dec.{i}.norm3")
    return out


def _assemble(cfg: ModelConfig, arrays: dict) -> Weights:
    proj = lambda w, b: Projection(np.asarray(arrays[w], np.float32), np.asarray(arrays[b], np.float32))
    norm = lambda p: NormParams(np.asarray(arrays[p + ".gain"], np.float32),
                                np.asarray(arrays[p + ".bias"], np.float32))

    def attn(p):
        return AttentionBlock(*(proj(f"{p}.{x}_w", f"{p}.{x}_b") for x in "qkvo"))

    enc = [EncoderLayer(attn(f"enc.{i}.attn"), norm(f"enc.{i}.norm1"),
                        FeedForward(proj(f"enc.{i}.ffn.w1", f"enc.{i}.ffn.b1"),
                                    proj(f"enc.{i}.ffn.w2", f"enc.{i}.ffn.b2")),
                        norm(f"enc.{i}.norm2")) for i in range(cfg.n_enc_layers)]
    dec = []
    for i in range(cfg.n_dec_layers):
        p = f"dec.{i}"
        has = cfg.ffn_dim_dec > 0
        dec.append(DecoderLayer(
            attn(f"{p}.self"), norm(f"{p}.norm1"), attn(f"{p}.cross"), norm(f"{p}.norm2"),
            FeedForward(proj(f"{p}.ffn.w1", f"{p}.ffn.b1"), proj(f"{p}.ffn.w2", f"{p}.ffn.b2"))
            if has else None,
            norm(f"{p}.norm3") if has else None))
    table = np.asarray(arrays["out_proj"], np.float32)
    return Weights(src_embed=np.asarray(arrays["src_embed"], np.float32),
                   tgt_embed=np.asarray(arrays["tgt_embed"], np.float32),
                   out_proj=Projection(table.T, np.asarray(arrays["out_bias"], np.float32)),
                   enc_layers=enc, dec_layers=dec,
                   positions=sinusoid_positions(cfg.max_positions, cfg.d_model))


def random_model(cfg: ModelConfig, seed: int) -> Weights:
    """Bit-identical to the reference's random_model(cfg, seed)."""
    cfg = config_of(cfg)
    gen = np.random.default_rng(seed)
    std = 1.0 / math.sqrt(cfg.d_model)
    arrays: dict[str, np.ndarray] = {}
    arrays["src_embed"] = (gen.standard_normal((cfg.vocab_size, cfg.d_model)) * std).astype(np.float32)
    for name in ("tgt_embed", "out_proj"):
        arrays[name] = arrays["src_embed"] if cfg.shared_embeddings else (
            gen.standard_normal((cfg.vocab_size, cfg.d_model)) * std).astype(np.float32)
    arrays["out_bias"] = (gen.standard_normal((cfg.vocab_size,)) * 0.01).astype(np.float32)
    for name, kind, shape in tensor_manifest(cfg):
        if name in arrays:
            continue
        if kind == "gemm":
            arrays[name] = (gen.standard_normal(shape) * std).astype(np.float32)
        elif name.endswith(".gain"):
            arrays[name] = (1.0 + 0.01 * gen.standard_normal(shape[0])).astype(np.float32)
        else:
            arrays[name] = (gen.standard_normal(shape) * 0.01).astype(np.float32)
    return _assemble(cfg, arrays)


def iter_named_tensors(cfg: ModelConfig, w, skip_gemm: bool = False
                       ) -> Iterator[tuple[str, np.ndarray]]:
    """(manifest name, float32 array) pairs of a Weights-like object, in the
    reference orientation (gemm weights [k, n]; out_proj as its [vocab, d]
    table).  Works for the reference's Weights too (duck-typed).  With
    ``skip_gemm`` the GEMM weights (and an unshared out_proj) are left out —
    the int8 upload sends those quantized (quant8.iter_quantized)."""
    yield "src_embed", np.asarray(w.src_embed, np.float32)
    if not cfg.shared_embeddings:
        yield "tgt_embed", np.asarray(w.tgt_embed, np.float32)
        if not skip_gemm:
            yield "out_proj", np.asarray(w.out_proj.weight, np.float32).T
    yield "out_bias", np.asarray(w.out_proj.bias, np.float32)

    def block(prefix, blk):
        for part in "qkvo":
            pr = getattr(blk, part)
            if not skip_gemm:
                yield f"{prefix}.{part}_w", np.asarray(pr.weight, np.float32)
            yield f"{prefix}.{part}_b", np.asarray(pr.bias, np.float32)

    def norm(prefix, n):
        yield f"{prefix}.gain", np.asarray(n.gain, np.float32)
        yield f"{prefix}.bias", np.asarray(n.bias, np.float32)

    def ffn(prefix, f):
        for wn, bn, pr in (("w1", "b1", f.w1), ("w2", "b2", f.w2)):
            if not skip_gemm:
                yield f"{prefix}.{wn}", np.asarray(pr.weight, np.float32)
            yield f"{prefix}.{bn}", np.asarray(pr.bias, np.float32)

    for i, L in enumerate(w.enc_layers):
        yield from block(f"enc.{i}.attn", L.attn)
        yield from norm(f"enc.{i}.norm1", L.norm1)
        yield from ffn(f"enc.{i}.ffn", L.ffn)
        yield from norm(f"enc.{i}.norm2", L.norm2)
    for i, L in enumerate(w.dec_layers):
        yield from block(f"dec.{i}.self", L.self_attn)
        yield from norm(f"dec.{i}.norm1", L.norm1)
        yield from block(f"dec.{i}.cross", L.cross_attn)
        yield from norm(f"dec.{i}.norm2", L.norm2)
        if L.ffn is not None:
            yield from ffn(f"dec.{i}.ffn", L.ffn)
            yield from norm(f"dec.{i}.norm3", L.norm3)
    if getattr(w, "positions", None) is not None:
        yield "positions", np.asarray(w.positions, np.float32)
