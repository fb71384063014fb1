"""CPU oracle for the B200 translation engine — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference `fastnmt` hot path
(model construction -> encoder -> incremental decoder -> greedy / beam search
-> length-sorted batching).  It exists so the CUDA engine in
``paper_2109_08003_b200`` can be checked bit-for-bit / within tolerance
against the reference semantics without importing the reference at test time
(the reference tree does not exist on the GPU box).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module.  The product package never does.

Parity status: PINNED.  ``oracle/make_golden.py`` ran the unmodified
reference (``/root/reference/pkg/src/fastnmt``) in the build container and
committed its outputs under ``tests/golden/``; ``tests/test_oracle_golden.py``
checks this restatement against them bit-for-bit (same numpy einsum order).

Layout differs on purpose from the reference: parameters live in one flat
``dict[name -> np.ndarray]`` keyed by the reference's tensor-manifest names
(store.py:88-115), weights stay in the reference ``[k, n]`` orientation
(x @ W), and the decoder cache is a plain dict.

Citations (reference file:line, relative to /root/reference/pkg/src/fastnmt):
  tensor.py:46-134  matmul / rowsum / softmax / norms / relu
  model.py:45-70    ModelConfig validation
  model.py:184-190  interleaved sinusoid table
  model.py:199-245  attention, additive mask
  model.py:261-344  encode, init_cross_cache, decode_step
  model.py:347-367  count_params
  search.py:49-147  max_out_length, greedy_translate, beam_translate
  batching.py:68-165 plan_batches, restore_order, estimate_peak_memory
  store.py:88-115, 539-572  manifest order and random_model RNG draws
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

PAD, UNK, BOS, EOS = 0, 1, 2, 3          # textpipe.py:43-45
MASK_VALUE = np.float32(-1e9)            # model.py:37-38
NORM_EPS = np.float32(1e-6)              # tensor.py:34


# ----------------------------------------------------------------------------
# configuration (model.py:45-70)

@dataclass(frozen=True)
class Arch:
    n_enc_layers: int
    n_dec_layers: int
    d_model: int
    n_heads_enc: int
    n_heads_dec: int
    ffn_dim_enc: int
    ffn_dim_dec: int
    vocab_size: int
    max_positions: int
    norm_variant: str = "l2"
    shared_embeddings: bool = True

    def __post_init__(self):
        sizes = (self.n_enc_layers, self.n_dec_layers, self.d_model, self.n_heads_enc,
                 self.n_heads_dec, self.ffn_dim_enc, self.vocab_size, self.max_positions)
        if any(s < 1 for s in sizes) or self.ffn_dim_dec < 0:
            raise ValueError("invalid sizes")
        if self.d_model % self.n_heads_enc or self.d_model % self.n_heads_dec:
            raise ValueError("heads must divide d_model")
        if self.norm_variant not in ("l2", "l1"):
            raise ValueError("bad norm variant")


def arch_of(cfg) -> Arch:
    """Accept any object with the ModelConfig field names."""
    return Arch(**{f: getattr(cfg, f) for f in Arch.__dataclass_fields__})


def param_count(a: Arch) -> int:
    """model.py:347-367 — embeddings once if shared, else three tables."""
    d = a.d_model
    lin = lambda i, o: i * o + o
    enc = 4 * lin(d, d) + lin(d, a.ffn_dim_enc) + lin(a.ffn_dim_enc, d) + 4 * d
    dec = 8 * lin(d, d) + 4 * d
    if a.ffn_dim_dec:
        dec += lin(d, a.ffn_dim_dec) + lin(a.ffn_dim_dec, d) + 2 * d
    emb = a.vocab_size * d * (1 if a.shared_embeddings else 3)
    return emb + a.vocab_size + a.n_enc_layers * enc + a.n_dec_layers * dec


# ----------------------------------------------------------------------------
# construction (store.py:88-115 manifest order, store.py:539-572 draws)

def manifest(a: Arch):
    """(name, kind, shape) in the reference's draw order."""
    d, v = a.d_model, a.vocab_size
    out = [("src_embed", "embed", (v, d)), ("tgt_embed", "embed", (v, d)),
           ("out_proj", "out_proj", (v, d)), ("out_bias", "plain", (v,))]

    def attn(p):
        for part in "qkvo":
            out.append((f"{p}.{part}_w", "gemm", (d, d)))
            out.append((f"{p}.{part}_b", "plain", (d,)))

    def norm(p):
        out.append((f"{p}.gain", "plain", (d,)))
        out.append((f"{p}.bias", "plain", (d,)))

    def ffn(p, f):
        out.extend([(f"{p}.w1", "gemm", (d, f)), (f"{p}.b1", "plain", (f,)),
                    (f"{p}.w2", "gemm", (f, d)), (f"{p}.b2", "plain", (d,))])

    for i in range(a.n_enc_layers):
        attn(f"enc.{i}.attn"); norm(f"enc.{i}.norm1")
        ffn(f"enc.{i}.ffn", a.ffn_dim_enc); norm(f"enc.{i}.norm2")
    for i in range(a.n_dec_layers):
        attn(f"dec.{i}.self"); norm(f"dec.{i}.norm1")
        attn(f"dec.{i}.cross"); norm(f"dec.{i}.norm2")
        if a.ffn_dim_dec > 0:
            ffn(f"dec.{i}.ffn", a.ffn_dim_dec); norm(f"dec.{i}.norm3")
    return out


def make_params(a: Arch, seed: int) -> dict:
    """Same PCG64 stream and draw order as store.random_model.

    Returns name -> float32 array.  ``out_proj`` is stored [vocab, d] (the
    reference transposes it at assembly, store.py:195-202); with shared
    embeddings the three tables are one array.
    """
    g = np.random.default_rng(seed)
    s = 1.0 / math.sqrt(a.d_model)
    dense = lambda shape: (g.standard_normal(shape) * s).astype(np.float32)
    tiny = lambda shape: (g.standard_normal(shape) * 0.01).astype(np.float32)
    p = {"src_embed": dense((a.vocab_size, a.d_model))}
    p["tgt_embed"] = p["src_embed"] if a.shared_embeddings else dense((a.vocab_size, a.d_model))
    p["out_proj"] = p["src_embed"] if a.shared_embeddings else dense((a.vocab_size, a.d_model))
    p["out_bias"] = tiny((a.vocab_size,))
    for name, kind, shape in manifest(a):
        if name in p:
            continue
        if kind == "gemm":
            p[name] = dense(shape)
        elif name.endswith(".gain"):
            p[name] = (1.0 + 0.01 * g.standard_normal(shape[0])).astype(np.float32)
        else:
            p[name] = tiny(shape)
    p["positions"] = position_table(a.max_positions, a.d_model)
    return p


def params_from_weights(a: Arch, w) -> dict:
    """Flatten a reference-style ``Weights`` object (duck-typed) into the dict."""
    p = {"src_embed": np.asarray(w.src_embed, np.float32),
         "tgt_embed": np.asarray(w.tgt_embed, np.float32),
         "out_proj": np.asarray(w.out_proj.weight, np.float32).T,
         "out_bias": np.asarray(w.out_proj.bias, np.float32),
         "positions": np.asarray(w.positions, np.float32)}

    def put_attn(prefix, blk):
        for part in "qkvo":
            proj = getattr(blk, part)
            p[f"{prefix}.{part}_w"] = np.asarray(proj.weight, np.float32)
            p[f"{prefix}.{part}_b"] = np.asarray(proj.bias, np.float32)

    def put_norm(prefix, n):
        p[f"{prefix}.gain"] = np.asarray(n.gain, np.float32)
        p[f"{prefix}.bias"] = np.asarray(n.bias, np.float32)

    def put_ffn(prefix, f):
        p[f"{prefix}.w1"], p[f"{prefix}.b1"] = np.asarray(f.w1.weight), np.asarray(f.w1.bias)
        p[f"{prefix}.w2"], p[f"{prefix}.b2"] = np.asarray(f.w2.weight), np.asarray(f.w2.bias)

    for i, L in enumerate(w.enc_layers):
        put_attn(f"enc.{i}.attn", L.attn); put_norm(f"enc.{i}.norm1", L.norm1)
        put_ffn(f"enc.{i}.ffn", L.ffn); put_norm(f"enc.{i}.norm2", L.norm2)
    for i, L in enumerate(w.dec_layers):
        put_attn(f"dec.{i}.self", L.self_attn); put_norm(f"dec.{i}.norm1", L.norm1)
        put_attn(f"dec.{i}.cross", L.cross_attn); put_norm(f"dec.{i}.norm2", L.norm2)
        if L.ffn is not None:
            put_ffn(f"dec.{i}.ffn", L.ffn); put_norm(f"dec.{i}.norm3", L.norm3)
    return p


def position_table(n_pos: int, d: int) -> np.ndarray:
    """model.py:184-190: sin on even columns, cos on odd, angle uses 2*floor(i/2)."""
    i = np.arange(d, dtype=np.float64)
    inv = np.power(10000.0, (2.0 * np.floor(i / 2.0)) / d)
    ang = np.arange(n_pos, dtype=np.float64)[:, None] / inv[None, :]
    tab = np.where((np.arange(d) % 2 == 0)[None, :], np.sin(ang), np.cos(ang))
    return tab.astype(np.float32)


# ----------------------------------------------------------------------------
# primitive kernels (tensor.py:46-134)

def mm(x, w):
    """In-order accumulation einsum (tensor.py:57); batch-row invariant."""
    return np.einsum("ik,kj->ij", x, w)


def ordered_sum(x):
    return np.einsum("...k->...", x)


def softmax_last(x):
    e = np.exp(x - x.max(axis=-1, keepdims=True))
    return e / ordered_sum(e)[..., None]


def norm_rows(variant: str, x, gain, bias):
    """tensor.py:84-129 (f64 row mean; eps added to the deviation scale)."""
    mu = x.mean(axis=-1, keepdims=True, dtype=np.float64).astype(np.float32)
    dev = x - mu
    if variant == "l1":
        scale = np.abs(dev).mean(axis=-1, keepdims=True)
    else:
        scale = np.sqrt(np.square(dev).mean(axis=-1, keepdims=True))
    return gain * dev / (scale + NORM_EPS) + bias


def linear(p, wname, bname, x2d):
    return mm(x2d, p[wname]) + p[bname]


def linear3(p, wname, bname, x3d):
    b, l, _ = x3d.shape
    return linear(p, wname, bname, x3d.reshape(b * l, -1)).reshape(b, l, -1)


def mha(q, k, v, add_mask, heads: int):
    """model.py:199-240: scale the query, 1-head path skips the reshape."""
    b, lq, d = q.shape
    lk = k.shape[1]
    dk = d // heads
    qs = q * np.float32(1.0 / math.sqrt(dk))
    if heads == 1:
        s = np.einsum("bqd,bkd->bqk", qs, k)
        if add_mask is not None:
            s = s + add_mask
        return np.einsum("bqk,bkd->bqd", softmax_last(s), v)
    s = np.einsum("bqhd,bkhd->bhqk", qs.reshape(b, lq, heads, dk), k.reshape(b, lk, heads, dk))
    if add_mask is not None:
        s = s + add_mask[:, None, :, :]
    o = np.einsum("bhqk,bkhd->bqhd", softmax_last(s), v.reshape(b, lk, heads, dk))
    return np.ascontiguousarray(o).reshape(b, lq, d)


def key_mask(valid):
    return np.where(np.asarray(valid, bool)[:, None, :], np.float32(0), MASK_VALUE)


# ----------------------------------------------------------------------------
# encoder / decoder (model.py:261-344)

def encoder(a: Arch, p: dict, tokens, valid):
    """Returns states f32 [b, s, d]; pad rows are computed like the reference."""
    tokens = np.asarray(tokens)
    if tokens.size and (tokens.min() < 0 or tokens.max() >= a.vocab_size):
        raise ValueError("token id out of range")
    b, s = tokens.shape
    if s > a.max_positions:
        raise OverflowError("source longer than max_positions")
    x = p["src_embed"][tokens] * np.float32(math.sqrt(a.d_model))
    x = x + p["positions"][:s]
    m = key_mask(valid)
    for i in range(a.n_enc_layers):
        pre = f"enc.{i}"
        q = linear3(p, f"{pre}.attn.q_w", f"{pre}.attn.q_b", x)
        k = linear3(p, f"{pre}.attn.k_w", f"{pre}.attn.k_b", x)
        v = linear3(p, f"{pre}.attn.v_w", f"{pre}.attn.v_b", x)
        att = mha(q, k, v, m, a.n_heads_enc)
        x = norm_rows(a.norm_variant, x + linear3(p, f"{pre}.attn.o_w", f"{pre}.attn.o_b", att),
                      p[f"{pre}.norm1.gain"], p[f"{pre}.norm1.bias"])
        h = np.maximum(linear(p, f"{pre}.ffn.w1", f"{pre}.ffn.b1", x.reshape(b * s, -1)),
                       np.float32(0))
        h = linear(p, f"{pre}.ffn.w2", f"{pre}.ffn.b2", h).reshape(b, s, -1)
        x = norm_rows(a.norm_variant, x + h, p[f"{pre}.norm2.gain"], p[f"{pre}.norm2.bias"])
    return x


def start_cache(a: Arch, p: dict, states, valid) -> dict:
    """model.py:290-305: cross K/V once per decoder layer; empty self history."""
    b, s, d = states.shape
    c = {"t": 0, "mask": key_mask(valid), "self_k": [], "self_v": [], "cross_k": [], "cross_v": []}
    for i in range(a.n_dec_layers):
        c["cross_k"].append(linear3(p, f"dec.{i}.cross.k_w", f"dec.{i}.cross.k_b", states))
        c["cross_v"].append(linear3(p, f"dec.{i}.cross.v_w", f"dec.{i}.cross.v_b", states))
        c["self_k"].append(np.zeros((b, 0, d), np.float32))
        c["self_v"].append(np.zeros((b, 0, d), np.float32))
    return c


def pick_rows(c: dict, rows) -> dict:
    """model.py:170-181 beam reorder (cross K/V and mask gathered too)."""
    idx = np.asarray(rows, dtype=np.intp)
    out = {"t": c["t"], "mask": c["mask"][idx]}
    for key in ("self_k", "self_v", "cross_k", "cross_v"):
        out[key] = [arr[idx] for arr in c[key]]
    return out


def decoder_step(a: Arch, p: dict, c: dict, prev) -> np.ndarray:
    """model.py:308-344 — raw logits f32 [b, vocab]; mutates the cache."""
    prev = np.asarray(prev)
    if prev.size and (prev.min() < 0 or prev.max() >= a.vocab_size):
        raise ValueError("token id out of range")
    t = c["t"]
    if t >= a.max_positions:
        raise OverflowError("decode position beyond max_positions")
    b = prev.shape[0]
    x = p["tgt_embed"][prev] * np.float32(math.sqrt(a.d_model))
    x = (x + p["positions"][t]).reshape(b, 1, -1)
    nv, h = a.norm_variant, a.n_heads_dec
    for i in range(a.n_dec_layers):
        pre = f"dec.{i}"
        q = linear3(p, f"{pre}.self.q_w", f"{pre}.self.q_b", x)
        k = linear3(p, f"{pre}.self.k_w", f"{pre}.self.k_b", x)
        v = linear3(p, f"{pre}.self.v_w", f"{pre}.self.v_b", x)
        c["self_k"][i] = np.concatenate([c["self_k"][i], k], axis=1)
        c["self_v"][i] = np.concatenate([c["self_v"][i], v], axis=1)
        att = mha(q, c["self_k"][i], c["self_v"][i], None, h)
        x = norm_rows(nv, x + linear3(p, f"{pre}.self.o_w", f"{pre}.self.o_b", att),
                      p[f"{pre}.norm1.gain"], p[f"{pre}.norm1.bias"])
        qc = linear3(p, f"{pre}.cross.q_w", f"{pre}.cross.q_b", x)
        att = mha(qc, c["cross_k"][i], c["cross_v"][i], c["mask"], h)
        x = norm_rows(nv, x + linear3(p, f"{pre}.cross.o_w", f"{pre}.cross.o_b", att),
                      p[f"{pre}.norm2.gain"], p[f"{pre}.norm2.bias"])
        if a.ffn_dim_dec > 0:
            hid = np.maximum(linear(p, f"{pre}.ffn.w1", f"{pre}.ffn.b1", x.reshape(b, -1)),
                             np.float32(0))
            y = linear(p, f"{pre}.ffn.w2", f"{pre}.ffn.b2", hid).reshape(b, 1, -1)
            x = norm_rows(nv, x + y, p[f"{pre}.norm3.gain"], p[f"{pre}.norm3.bias"])
    c["t"] = t + 1
    return mm(x.reshape(b, -1), p["out_proj"].T) + p["out_bias"]


# ----------------------------------------------------------------------------
# search (search.py:49-147)

def out_budget(src_len: int, max_positions: int, ratio: float = 1.5, offset: int = 5) -> int:
    return max(1, min(max_positions, math.ceil(ratio * src_len) + offset))


def top2_of(logits):
    """Per row: (top-1 value, top-2 value, top-2 id); top-1 is np.argmax's
    lowest-id maximum (search.py:71), top-2 the best of the rest."""
    rows = np.arange(logits.shape[0])
    i1 = np.argmax(logits, axis=1)
    v1 = logits[rows, i1].copy()
    rest = logits.copy()
    rest[rows, i1] = -np.inf
    i2 = np.argmax(rest, axis=1)
    return v1, rest[rows, i2].copy(), i2.astype(np.int32)


def greedy(a: Arch, p: dict, tokens, valid, ratio=1.5, offset=5, bos=BOS, eos=EOS, pad=PAD,
           trace=None):
    """search.py:58-86.  Returns list of id lists (no BOS/EOS).

    ``trace`` (a list) receives one ``top2_of`` triple per step (all rows), the
    near-tie evidence for the fp16/bf16 parity reports."""
    valid = np.asarray(valid, bool)
    n = valid.shape[0]
    if n == 0:
        return []
    states = encoder(a, p, tokens, valid)
    budget = [out_budget(int(s), a.max_positions, ratio, offset) for s in valid.sum(axis=1)]
    c = start_cache(a, p, states, valid)
    feed = np.full(n, bos, np.int64)
    done = np.zeros(n, bool)
    res = [[] for _ in range(n)]
    for t in range(max(budget)):
        logits = decoder_step(a, p, c, feed)
        best = np.argmax(logits, axis=1)
        if trace is not None:
            trace.append(top2_of(logits))
        feed = np.full(n, pad, np.int64)
        for r in np.flatnonzero(~done):
            tok = int(best[r])
            if tok == eos:
                done[r] = True
                continue
            res[r].append(tok)
            feed[r] = tok
            done[r] = t + 1 >= budget[r]
        if done.all():
            break
    return res


def log_softmax64(logits):
    """search.py:89-91 (float64)."""
    z = logits - logits.max(axis=-1, keepdims=True)
    return z - np.log(ordered_sum(np.exp(z)))[..., None]


def beam_sentence(a: Arch, p: dict, states_row, valid_row, k: int,
                  ratio=1.5, offset=5, bos=BOS, eos=EOS, trace=None, trace_width=None):
    """search.py:114-147 for one sentence (states_row [1,s,d]).

    Candidate order is (score desc, token asc, parent asc); an EOS pick moves
    the hypothesis to the finished pool and still consumes one of the k slots.
    Returns (tokens, score, finished).

    ``trace`` (a list) receives, per step, the first ``trace_width`` (default
    3k) candidates in that order as (score f64, token, parent) arrays: enough
    to replay the search and to measure how close any other hypothesis came
    to being kept (the near-tie report of the GPU beam parity tests).
    """
    limit = out_budget(int(np.asarray(valid_row).sum()), a.max_positions, ratio, offset)
    c = start_cache(a, p, states_row, valid_row)
    live = [((), 0.0)]
    fin = []
    for _ in range(limit):
        feed = np.array([h[0][-1] if h[0] else bos for h in live], np.int64)
        lp = log_softmax64(decoder_step(a, p, c, feed).astype(np.float64))
        # Exact same ordering as the reference's python sort, via lexsort on
        # (parent, token, -score): primary key is the last one given.
        sc = np.array([h[1] for h in live])[:, None] + lp
        par = np.repeat(np.arange(len(live)), lp.shape[1])
        tok = np.tile(np.arange(lp.shape[1]), len(live))
        flat = sc.reshape(-1)
        # python float addition == numpy float64 addition (both IEEE binary64)
        if trace is not None:
            wide = np.lexsort((par, tok, -flat))[:trace_width or 3 * k]
            trace.append((flat[wide].astype(np.float64), tok[wide].astype(np.int32),
                          par[wide].astype(np.int32)))
            order = wide[:k]
        else:
            order = np.lexsort((par, tok, -flat))[:k]
        nxt, parents = [], []
        for j in order:
            sj, tj, pj = float(flat[j]), int(tok[j]), int(par[j])
            if tj == eos:
                fin.append((live[pj][0], sj))
            else:
                nxt.append((live[pj][0] + (tj,), sj))
                parents.append(pj)
        live = nxt
        if not live or len(fin) >= k:
            break
        c = pick_rows(c, parents)
    if fin:
        pool, finished = fin, True
    else:
        pool, finished = live, False
    best = max(pool, key=lambda h: (h[1], tuple(-x for x in h[0])))
    return list(best[0]), best[1], finished


def beam_divergence(steps, k: int, hyp, budget: int, eos=EOS):
    """Near-tie measure for a beam output ``hyp`` that differs from the
    oracle's.  ``steps`` is a ``beam_sentence`` trace (per step: candidate
    scores / tokens / parents in the reference's sort order, search.py:125-127).

    Replays the whole oracle search and returns (where, step, gap) with gap
    the smaller of the two score margins that can explain the divergence:
      * "hyp": at the first step the oracle did not keep hyp's extension, the
        oracle's k-th kept score minus hyp's candidate score (inf when it is
        outside the traced width); if hyp survived to the end, the oracle's
        best final score minus hyp's (search.py:145-147);
      * "best": the smallest margin by which the oracle's best hypothesis
        stayed inside the beam (its candidate's score minus the first pruned
        candidate's) — a search that dropped it had its ranking flipped there.
    ``hyp`` finished with EOS iff len(hyp) < budget (search.py:116-140).
    """
    hyp = tuple(int(x) for x in hyp)
    finished = len(hyp) < budget
    live, fin = [((), 0.0)], []
    kept_log = []            # per step: {(tokens, finished?): (score, margin)}
    hyp_gap = hyp_where = None
    for t, (sc, tok, par) in enumerate(steps):
        nxt_score = float(sc[k]) if len(sc) > k else float("-inf")
        kept, nxt = {}, []
        for j in range(min(k, len(tok))):
            pj, tj, sj = int(par[j]), int(tok[j]), float(sc[j])
            if tj == eos:
                fin.append((live[pj][0], sj))
                kept[(live[pj][0], True)] = (sj, sj - nxt_score)
            else:
                nxt.append((live[pj][0] + (tj,), sj))
                kept[(live[pj][0] + (tj,), False)] = (sj, sj - nxt_score)
        kept_log.append(kept)
        if hyp_gap is None and (t < len(hyp) or (finished and t == len(hyp))):
            key = (hyp, True) if t == len(hyp) else (hyp[:t + 1], False)
            if key not in kept:
                prefix = hyp[:t]
                pidx = next((i for i, h in enumerate(live) if h[0] == prefix), None)
                want = hyp[t] if t < len(hyp) else eos
                hit = [j for j in range(len(tok))
                       if pidx is not None and int(tok[j]) == want and int(par[j]) == pidx]
                hyp_gap = float(sc[k - 1] - sc[hit[0]]) if hit else float("inf")
                hyp_where = t
        live = nxt
        if not live or len(fin) >= k:
            break
    pool = fin if fin else live
    best = max(pool, key=lambda h: (h[1], tuple(-x for x in h[0])))
    if hyp_gap is None:
        mine = [h for h in pool if h[0] == hyp]
        hyp_gap = float(best[1] - mine[0][1]) if mine else float("inf")
        hyp_where = len(kept_log) - 1
    margins = []
    for t, kept in enumerate(kept_log):
        if t < len(best[0]):
            key = (best[0][:t + 1], False)
        elif fin and t == len(best[0]):
            key = (best[0], True)
        else:
            break
        if key in kept:
            margins.append((kept[key][1], t))
    best_gap, best_t = min(margins) if margins else (float("inf"), -1)
    if best_gap < hyp_gap:
        return ("best", best_t, float(best_gap))
    return ("hyp", hyp_where, float(hyp_gap))


def greedy_divergence(ref, got, top1, top2, top2_id):
    """First divergent step of a greedy output and the reference's top-1 minus
    top-2 logit gap there (inf if ``got`` took a token other than the
    reference's runner-up).  top*/top2_id are the reference's per-step values
    for this sentence.  Returns None when the outputs are identical."""
    ref, got = list(ref), list(got)
    if ref == got:
        return None
    j = next((i for i in range(min(len(ref), len(got))) if ref[i] != got[i]),
             min(len(ref), len(got)))
    if j >= len(top1):
        return (j, float("inf"))
    alt = got[j] if j < len(got) else EOS
    gap = float(top1[j] - top2[j]) if int(top2_id[j]) == alt else float("inf")
    return (j, gap)


def beam(a: Arch, p: dict, tokens, valid, k: int, ratio=1.5, offset=5):
    valid = np.asarray(valid, bool)
    states = encoder(a, p, tokens, valid)
    return [beam_sentence(a, p, states[i:i + 1], valid[i:i + 1], k, ratio, offset)[0]
            for i in range(valid.shape[0])]


# ----------------------------------------------------------------------------
# batching (batching.py:68-165)

def length_order(lengths):
    """Stable descending sort (batching.py:68-70)."""
    return sorted(range(len(lengths)), key=lambda i: -lengths[i])


def group_sorted(sorted_lengths, sbatch: int, wbatch: int):
    """batching.py:73-97 -> list of (positions, max_len, oversize)."""
    groups, cur, top = [], [], 0
    for pos, n in enumerate(sorted_lengths):
        if cur and len(cur) + 1 <= sbatch and (len(cur) + 1) * top <= wbatch:
            cur.append(pos)
            continue
        if cur:
            groups.append((cur, top, top > wbatch))
        cur, top = [pos], n
    if cur:
        groups.append((cur, top, top > wbatch))
    return groups


def plan(lengths, sbatch: int, wbatch: int):
    """batching.py:100-109 -> (list of (indices, max_len, oversize), permutation)."""
    order = length_order(lengths)
    groups = group_sorted([lengths[i] for i in order], sbatch, wbatch)
    batches = [([order[q] for q in g], top, over) for g, top, over in groups]
    perm = [i for b in batches for i in b[0]]
    return batches, perm


def unpermute(outputs, perm):
    """batching.py:112-122."""
    if len(outputs) != len(perm):
        raise ValueError("output count does not match the plan")
    res = [None] * len(perm)
    for o, i in zip(outputs, perm):
        res[i] = o
    return res


def peak_bytes(batches, a: Arch, max_out_len: int) -> int:
    """batching.py:134-165 (f32 accounting, 8 MiB base, 1.5x slack)."""
    base = 8 << 20
    if not batches:
        return base
    n_max = max(len(b[0]) for b in batches)
    nl = max(len(b[0]) * b[1] for b in batches)
    nll = max(len(b[0]) * b[1] * b[1] for b in batches)
    ncache = max(len(b[0]) * (b[1] + max_out_len) for b in batches)
    d = a.d_model
    heads = max(a.n_heads_enc, a.n_heads_dec)
    ffn = max(a.ffn_dim_enc, a.ffn_dim_dec, d)
    live = (nl * d + nl * d * (a.n_enc_layers + 4) + nll * heads * 3 + nl * ffn * 2
            + ncache * d * a.n_dec_layers * 2 + n_max * a.vocab_size * 2) * 4
    return base + math.ceil(1.5 * live)


# ----------------------------------------------------------------------------
# synthetic workloads

STUDENT_6_1_1 = Arch(6, 1, 512, 1, 1, 2048, 2048, 32772, 1024)
STUDENT_6_1_8 = Arch(6, 1, 512, 8, 8, 2048, 2048, 32772, 1024)
STUDENT_6_6_8 = Arch(6, 6, 512, 8, 8, 2048, 2048, 32772, 1024, shared_embeddings=False)
DEEP_12_768 = Arch(12, 6, 768, 8, 8, 3072, 3072, 32772, 1024)


def config1_sentences(n: int = 64, seed: int = 1234, vocab: int = 32772):
    """Config 1: lengths uniform in [10, 40], ids uniform in [4, vocab)."""
    g = np.random.default_rng(seed)
    lens = g.integers(10, 41, size=n)
    return [g.integers(4, vocab, size=int(L)).astype(np.int64) for L in lens]


def newstest_lengths(n: int, seed: int = 20211) -> np.ndarray:
    """clip(round(Gamma(3, 8)), 1, 200): mean ~24, p99 ~67 BPE tokens."""
    g = np.random.default_rng(seed)
    return np.clip(np.rint(g.gamma(3.0, 8.0, size=n)), 1, 200).astype(np.int32)


def pad_rows(rows, pad=PAD):
    n = len(rows)
    w = max((len(r) for r in rows), default=0)
    tok = np.full((n, w), pad, np.int64)
    valid = np.zeros((n, w), bool)
    for i, r in enumerate(rows):
        tok[i, :len(r)] = r
        valid[i, :len(r)] = True
    return tok, valid
