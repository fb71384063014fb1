"""Pin the CPU oracle (oracle/nmt_oracle.py) to the reference's own outputs,
frozen under tests/golden/ by oracle/make_golden.py.  Bit-exact where the
oracle issues the same numpy operations as the reference."""

import hashlib

import numpy as np
import pytest

from oracle import nmt_oracle as O


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, np.float32).tobytes()).hexdigest()


def test_known_answers(golden):
    g = golden("known_answers")
    assert np.array_equal(O.mm(g["mm_a"], g["mm_b"]), g["mm_out"])
    assert np.array_equal(g["mm_out"], np.array([[19, 22], [43, 50]], np.float32))
    assert np.array_equal(O.softmax_last(g["sm_in"]), g["sm_out"])
    assert np.allclose(g["sm_out"], [0.09003, 0.24473, 0.66524], atol=1e-5)
    assert np.array_equal(O.softmax_last(g["sm_big_in"]), g["sm_big_out"])
    for variant in ("l2", "l1"):
        got = O.norm_rows(variant, g["ln_in"], g["ln_gain"], g["ln_bias"])
        assert np.array_equal(got, g[f"ln_{variant}_out"])
        got = O.norm_rows(variant, g["ln_rand_in"], g["ln_rand_gain"], g["ln_rand_bias"])
        assert np.array_equal(got, g[f"ln_rand_{variant}"])
    # tensor.py:103-111 examples: [1,3] -> affine [-1,3]; constant row -> bias
    assert np.allclose(g["ln_l2_out"][0], [-1, 3], atol=1e-5)
    assert np.array_equal(g["ln_l2_out"][2], g["ln_bias"])
    pos = O.position_table(1024, 512)
    assert np.array_equal(pos[:64], g["positions_64x512"])
    assert sha(pos) == str(g["positions_1024x512_sha"])
    assert sha(O.position_table(1024, 768)) == str(g["positions_1024x768_sha"])
    for h in (1, 4):
        got = O.mha(g["att_q"], g["att_k"], g["att_v"], g["att_mask"], h)
        assert np.array_equal(got, g[f"att_h{h}"])


def _case_names(g):
    return sorted({k.split("__")[0] for k in g.files})


def _arch(cfg):
    c = [int(x) for x in cfg]
    return O.Arch(c[0], c[1], c[2], c[3], c[4], c[5], c[6], c[7], c[8],
                  norm_variant="l1" if c[9] else "l2", shared_embeddings=bool(c[10]))


def _split(ids, lens):
    out, o = [], 0
    for n in lens:
        out.append([int(x) for x in ids[o:o + n]])
        o += n
    return out


CASES = ["tiny", "tiny_dec2_h2", "tiny_noffn", "tiny_l1", "tiny_unshared", "d32_student",
         "d64_h8_dec6", "d64_h1_l1"]


@pytest.mark.parametrize("tag", CASES)
def test_small_models_bit_exact(golden, tag):
    g = golden("small_models")
    get = lambda k: g[f"{tag}__{k}"]
    a = _arch(get("config"))
    assert O.param_count(a) == int(get("count_params"))
    p = O.make_params(a, int(get("seed")))
    assert sha(p["src_embed"]) == str(get("src_embed_sha"))
    assert sha(p["enc.0.attn.q_w"]) == str(get("enc0_q_sha"))
    tok, valid = get("tokens"), get("valid")
    states = O.encoder(a, p, tok, valid)
    assert np.array_equal(states, get("states"))
    c = O.start_cache(a, p, states, valid)
    prev = np.full(tok.shape[0], O.BOS, np.int64)
    forced = get("forced")
    for t in range(6):
        assert np.array_equal(O.decoder_step(a, p, c, prev), get("logits")[t])
        prev = forced[:, t]
    assert O.greedy(a, p, tok, valid) == _split(get("greedy_ids"), get("greedy_lens"))
    for k in (1, 2, 4):
        assert O.beam(a, p, tok, valid, k) == _split(get(f"beam{k}_ids"), get(f"beam{k}_lens"))


def test_student_construction_pinned(golden):
    g = golden("students")
    archs = {"student_6_1_1": O.STUDENT_6_1_1, "student_6_1_8": O.STUDENT_6_1_8,
             "student_6_6_8": O.STUDENT_6_6_8, "deep_12_768": O.DEEP_12_768}
    for tag, a in archs.items():
        assert O.param_count(a) == int(g[f"{tag}_count"])
    assert int(g["student_6_1_1_count"]) == 39_930_372
    for tag in ("student_6_1_1", "student_6_6_8"):
        p = O.make_params(archs[tag], 0)
        assert sha(p["src_embed"]) == str(g[f"{tag}_src_embed_sha"])
        assert sha(p["tgt_embed"]) == str(g[f"{tag}_tgt_embed_sha"])
        assert sha(p["out_bias"]) == str(g[f"{tag}_out_bias_sha"])
        assert sha(p["dec.0.ffn.w2"]) == str(g[f"{tag}_dec0_ffn_w2_sha"])
        assert sha(p["enc.5.norm2.gain"]) == str(g[f"{tag}_enc5_norm2_gain_sha"])


def test_batching_matches_reference(golden):
    g = golden("batching")
    for i in range(6):
        lengths = [int(x) for x in g[f"c{i}_lengths"]]
        sb, wb = (int(x) for x in g[f"c{i}_caps"])
        batches, perm = O.plan(lengths, sb, wb)
        assert perm == [int(x) for x in g[f"c{i}_perm"]]
        assert [len(b[0]) for b in batches] == [int(x) for x in g[f"c{i}_sizes"]]
        assert [b[1] for b in batches] == [int(x) for x in g[f"c{i}_maxlen"]]
        assert [b[2] for b in batches] == [bool(x) for x in g[f"c{i}_oversize"]]
        assert O.unpermute(perm, perm) == list(range(len(lengths)))


def test_config1_inputs_match_recorded(golden):
    g = golden("config1_greedy")
    rows = O.config1_sentences()
    assert [len(r) for r in rows] == [int(x) for x in g["src_lens"]]
    assert np.array_equal(np.concatenate(rows), g["src_ids"])
    # random weights never emit EOS: every output runs to its budget
    budgets = [O.out_budget(len(r), 1024) for r in rows]
    assert [int(x) for x in g["out_lens"]] == budgets


@pytest.mark.slow
def test_config1_oracle_replays_reference():
    """Full Student-6-1-1 greedy over a 6-sentence slice (about 10 s)."""
    import numpy as np
    gz = np.load(__import__("conftest").GOLDEN / "config1_greedy.npz")
    rows = O.config1_sentences()[:6]
    p = O.make_params(O.STUDENT_6_1_1, 0)
    tok, valid = O.pad_rows(rows)
    got = O.greedy(O.STUDENT_6_1_1, p, tok, valid)
    want = _split(gz["out_ids"], gz["out_lens"])[:6]
    assert got == want
