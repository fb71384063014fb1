"""Generate the golden fixtures under tests/golden/ by running the UNMODIFIED
reference package (/root/reference/pkg/src/fastnmt) in the build container.

Test infrastructure only.  The reference cannot travel to the GPU box, so its
outputs are frozen here as small .npz fixtures; tests/test_oracle_golden.py
pins oracle/nmt_oracle.py against them and the GPU parity tests pin the CUDA
engine against the oracle and (for config 1) directly against the
reference's recorded greedy ids.

The reference's ``fastnmt/__init__.py`` imports ``fastnmt.engine`` which is
missing from the mounted tree; a stub module is registered in
``sys.modules`` first so the hot-path modules import.  No reference code is
copied.

Usage:  python oracle/make_golden.py [--skip-config1]
"""

from __future__ import annotations

import argparse
import hashlib
import sys
import time
import types
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def import_reference():
    if "fastnmt.engine" not in sys.modules:
        stub = types.ModuleType("fastnmt.engine")
        stub.RunConfig = type("RunConfig", (), {})
        stub.Translator = type("Translator", (), {})
        sys.modules["fastnmt.engine"] = stub
    sys.path.insert(0, str(REF_SRC))
    import fastnmt.batching as batching
    import fastnmt.model as model
    import fastnmt.search as search
    import fastnmt.store as store
    import fastnmt.tensor as tensor
    return types.SimpleNamespace(model=model, search=search, store=store, tensor=tensor,
                                 batching=batching)


TINY = dict(n_enc_layers=2, n_dec_layers=1, d_model=16, n_heads_enc=2, n_heads_dec=1,
            ffn_dim_enc=32, ffn_dim_dec=16, vocab_size=48, max_positions=64)

# (tag, overrides-on-TINY, seed): shapes drawn from the reference's own tests
# (tests/test_model.py:199-204, tests/test_acceptance.py:149-160).
SMALL_CASES = [
    ("tiny", {}, 30),
    ("tiny_dec2_h2", {"n_dec_layers": 2, "n_heads_dec": 2}, 31),
    ("tiny_noffn", {"ffn_dim_dec": 0}, 32),
    ("tiny_l1", {"norm_variant": "l1"}, 33),
    ("tiny_unshared", {"shared_embeddings": False, "n_heads_enc": 4}, 34),
    ("d32_student", {"n_enc_layers": 6, "d_model": 32, "n_heads_enc": 8, "n_heads_dec": 1,
                     "ffn_dim_enc": 128, "ffn_dim_dec": 32}, 35),
    ("d64_h8_dec6", {"n_enc_layers": 3, "n_dec_layers": 6, "d_model": 64, "n_heads_enc": 8,
                     "n_heads_dec": 8, "ffn_dim_enc": 256, "ffn_dim_dec": 256,
                     "vocab_size": 96}, 36),
    ("d64_h1_l1", {"n_enc_layers": 6, "d_model": 64, "n_heads_enc": 1, "n_heads_dec": 1,
                   "ffn_dim_enc": 256, "ffn_dim_dec": 256, "norm_variant": "l1"}, 37),
]

STUDENTS = {
    "student_6_1_1": dict(n_enc_layers=6, n_dec_layers=1, d_model=512, n_heads_enc=1,
                          n_heads_dec=1, ffn_dim_enc=2048, ffn_dim_dec=2048,
                          vocab_size=32772, max_positions=1024),
    "student_6_1_8": dict(n_enc_layers=6, n_dec_layers=1, d_model=512, n_heads_enc=8,
                          n_heads_dec=8, ffn_dim_enc=2048, ffn_dim_dec=2048,
                          vocab_size=32772, max_positions=1024),
    "student_6_6_8": dict(n_enc_layers=6, n_dec_layers=6, d_model=512, n_heads_enc=8,
                          n_heads_dec=8, ffn_dim_enc=2048, ffn_dim_dec=2048,
                          vocab_size=32772, max_positions=1024, shared_embeddings=False),
    "deep_12_768": dict(n_enc_layers=12, n_dec_layers=6, d_model=768, n_heads_enc=8,
                        n_heads_dec=8, ffn_dim_enc=3072, ffn_dim_dec=3072,
                        vocab_size=32772, max_positions=1024),
}


def sentences(rng, n, lo, hi, vocab):
    return [rng.integers(4, vocab, size=int(rng.integers(lo, hi + 1))) for _ in range(n)]


def padded(rows):
    w = max(len(r) for r in rows)
    tok = np.zeros((len(rows), w), np.int64)
    valid = np.zeros((len(rows), w), bool)
    for i, r in enumerate(rows):
        tok[i, :len(r)] = r
        valid[i, :len(r)] = True
    return tok, valid


def sha(arr) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr, np.float32).tobytes()).hexdigest()


def known_answers(ref) -> dict:
    t = ref.tensor
    f = lambda x: np.asarray(x, np.float32)
    rng = np.random.default_rng(3)
    out = {
        "mm_a": f([[1, 2], [3, 4]]), "mm_b": f([[5, 6], [7, 8]]),
        "mm_out": t.matmul(f([[1, 2], [3, 4]]), f([[5, 6], [7, 8]])),
        "sm_in": f([1, 2, 3]), "sm_out": t.softmax(f([1, 2, 3])),
        "sm_big_in": f([1000, 0]), "sm_big_out": t.softmax(f([1000, 0])),
        "ln_in": f([[1, 3], [10, 30], [5, 5]]),
        "ln_gain": f([2, 2]), "ln_bias": f([1, 1]),
    }
    out["ln_l2_out"] = t.layer_norm_l2(out["ln_in"], out["ln_gain"], out["ln_bias"])
    out["ln_l1_out"] = t.layer_norm_l1(out["ln_in"], out["ln_gain"], out["ln_bias"])
    x = f(rng.standard_normal((7, 40)) * 3 + 1)
    g, b = f(rng.standard_normal(40)), f(rng.standard_normal(40))
    out.update(ln_rand_in=x, ln_rand_gain=g, ln_rand_bias=b,
               ln_rand_l2=t.layer_norm_l2(x, g, b), ln_rand_l1=t.layer_norm_l1(x, g, b))
    pos = ref.model.sinusoid_positions(1024, 512)
    out["positions_64x512"] = pos[:64]
    out["positions_1024x512_sha"] = np.array(sha(pos))
    out["positions_1024x768_sha"] = np.array(sha(ref.model.sinusoid_positions(1024, 768)))
    q = f(rng.standard_normal((2, 3, 16)))
    k = f(rng.standard_normal((2, 5, 16)))
    v = f(rng.standard_normal((2, 5, 16)))
    mask = np.where(np.array([[1, 1, 1, 0, 0], [1, 1, 1, 1, 1]], bool)[:, None, :],
                    np.float32(0), np.float32(-1e9))
    out.update(att_q=q, att_k=k, att_v=v, att_mask=mask,
               att_h1=ref.model.attention(q, k, v, mask, 1),
               att_h4=ref.model.attention(q, k, v, mask, 4))
    return out


def small_case(ref, tag, overrides, seed) -> dict:
    M, S = ref.model, ref.search
    cfg = M.ModelConfig(**{**TINY, **overrides})
    w = ref.store.random_model(cfg, seed)
    tm = M.TranslationModel(cfg, w)
    rng = np.random.default_rng(seed + 1000)
    rows = sentences(rng, 5, 2, 9, cfg.vocab_size)
    tok, valid = padded(rows)
    enc = tm.encode(tok, valid)
    cache = tm.init_cache(enc)
    forced = rng.integers(4, cfg.vocab_size, size=(len(rows), 6))
    prev = np.full(len(rows), 2, np.int64)
    logits = []
    for t in range(6):
        logits.append(tm.step(cache, prev))
        prev = forced[:, t]
    sc = S.SearchConfig(bos_id=2, eos_id=3, pad_id=0)
    greedy = S.greedy_translate(tm, enc, sc)
    beams = {}
    for k in (1, 2, 4):
        sck = S.SearchConfig(bos_id=2, eos_id=3, pad_id=0, beam_size=k)
        beams[k] = S.beam_translate(tm, enc, sck)
    res = {
        "config": np.array([cfg.n_enc_layers, cfg.n_dec_layers, cfg.d_model, cfg.n_heads_enc,
                            cfg.n_heads_dec, cfg.ffn_dim_enc, cfg.ffn_dim_dec, cfg.vocab_size,
                            cfg.max_positions, int(cfg.norm_variant == "l1"),
                            int(cfg.shared_embeddings)], np.int64),
        "seed": np.array(seed), "tokens": tok, "valid": valid, "forced": forced,
        "states": enc.states, "logits": np.stack(logits),
        "count_params": np.array(M.count_params(cfg)),
        "src_embed_sha": np.array(sha(w.src_embed)),
        "enc0_q_sha": np.array(sha(w.enc_layers[0].attn.q.weight)),
    }
    for name, outs in [("greedy", greedy)] + [(f"beam{k}", v) for k, v in beams.items()]:
        flat = np.array([t for o in outs for t in o], np.int64)
        lens = np.array([len(o) for o in outs], np.int64)
        res[f"{name}_ids"], res[f"{name}_lens"] = flat, lens
    return res


def student_hashes(ref) -> dict:
    out = {}
    for tag, kw in STUDENTS.items():
        cfg = ref.model.ModelConfig(**kw)
        out[f"{tag}_count"] = np.array(ref.model.count_params(cfg))
        if tag in ("student_6_1_1", "student_6_6_8"):
            w = ref.store.random_model(cfg, 0)
            out[f"{tag}_src_embed_sha"] = np.array(sha(w.src_embed))
            out[f"{tag}_tgt_embed_sha"] = np.array(sha(w.tgt_embed))
            out[f"{tag}_out_bias_sha"] = np.array(sha(w.out_proj.bias))
            out[f"{tag}_dec0_ffn_w2_sha"] = np.array(sha(w.dec_layers[0].ffn.w2.weight))
            out[f"{tag}_enc5_norm2_gain_sha"] = np.array(sha(w.enc_layers[5].norm2.gain))
    return out


def batching_cases(ref) -> dict:
    B = ref.batching
    rng = np.random.default_rng(77)
    out = {}
    for i in range(6):
        n = int(rng.integers(0, 60))
        lengths = [int(x) for x in rng.integers(1, 300, size=n)]
        sb, wb = int(rng.integers(1, 16)), int(rng.integers(8, 800))
        plan = B.plan_batches(lengths, B.DecodeLimits(sbatch=sb, wbatch=wb))
        out[f"c{i}_lengths"] = np.array(lengths, np.int64)
        out[f"c{i}_caps"] = np.array([sb, wb], np.int64)
        out[f"c{i}_perm"] = np.array(plan.permutation, np.int64)
        out[f"c{i}_sizes"] = np.array([len(b.indices) for b in plan.batches], np.int64)
        out[f"c{i}_maxlen"] = np.array([b.max_len for b in plan.batches], np.int64)
        out[f"c{i}_oversize"] = np.array([b.oversize for b in plan.batches], bool)
    return out


def config1(ref) -> dict:
    """Student-6-1-1 greedy f32 over config 1's 64 sentences via the reference,
    recording per-step top-2 logits for the near-tie report."""
    M, S, B = ref.model, ref.search, ref.batching
    cfg = M.ModelConfig(**STUDENTS["student_6_1_1"])
    tm = M.TranslationModel(cfg, ref.store.random_model(cfg, 0))
    g = np.random.default_rng(1234)
    lens = g.integers(10, 41, size=64)
    rows = [g.integers(4, 32772, size=int(L)).astype(np.int64) for L in lens]
    sc = S.SearchConfig(bos_id=2, eos_id=3, pad_id=0)
    plan = B.plan_batches([len(r) for r in rows], B.DecodeLimits(sbatch=128, wbatch=2048))
    outs = []
    top1 = [None] * 64
    top2 = [None] * 64
    t0 = time.time()
    for batch in plan.batches:
        tok, valid = padded([rows[i] for i in batch.indices])
        enc = tm.encode(tok, valid)
        rec = []
        orig_step = tm.step

        class Recorder:
            max_positions = tm.max_positions
            init_cache = staticmethod(tm.init_cache)

            @staticmethod
            def step(cache, prev):
                lg = orig_step(cache, prev)
                part = np.partition(lg, -2, axis=1)[:, -2:]
                rec.append((part.max(axis=1), part.min(axis=1)))
                return lg

        o = S.greedy_translate(Recorder, enc, sc)
        outs.extend(o)
        for j, i in enumerate(batch.indices):
            top1[i] = np.array([r[0][j] for r in rec], np.float32)
            top2[i] = np.array([r[1][j] for r in rec], np.float32)
    outs = B.restore_order(outs, plan)
    print(f"config1 reference greedy: {time.time() - t0:.1f}s", file=sys.stderr)
    return {
        "src_lens": lens.astype(np.int64),
        "src_ids": np.concatenate(rows),
        "out_lens": np.array([len(o) for o in outs], np.int64),
        "out_ids": np.array([t for o in outs for t in o], np.int64),
        "top1": np.concatenate(top1), "top2": np.concatenate(top2),
        "step_counts": np.array([len(x) for x in top1], np.int64),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-config1", action="store_true")
    args = ap.parse_args()
    ref = import_reference()
    OUT.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(OUT / "known_answers.npz", **known_answers(ref))
    cases = {}
    for tag, ov, seed in SMALL_CASES:
        for k, v in small_case(ref, tag, ov, seed).items():
            cases[f"{tag}__{k}"] = v
    np.savez_compressed(OUT / "small_models.npz", **cases)
    np.savez_compressed(OUT / "students.npz", **student_hashes(ref))
    np.savez_compressed(OUT / "batching.npz", **batching_cases(ref))
    if not args.skip_config1:
        np.savez_compressed(OUT / "config1_greedy.npz", **config1(ref))
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
