"""CPU tests: the C-ABI library loads and exports the header, host-side
construction / scheduling / search logic matches the reference semantics."""

import hashlib
import math
import re
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import pytest

from oracle import nmt_oracle as O
from paper_2109_08003_b200 import batching as B
from paper_2109_08003_b200 import store as S

ROOT = Path(__file__).resolve().parent.parent


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, np.float32).tobytes()).hexdigest()


# --- C ABI -------------------------------------------------------------------

def header_functions():
    text = (ROOT / "include" / "fnmt_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fnmt_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_function():
    from paper_2109_08003_b200 import _capi
    names = header_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(_capi.lib, name), name
        assert name in _capi.EXPORTED, f"{name} has no ctypes signature"
    assert _capi.lib.fnmt_version().startswith(b"fnmt_b200")


def test_library_is_sm100a_cubin():
    import subprocess
    so = ROOT / "paper_2109_08003_b200" / "libfnmt_b200.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_capi_rejects_bad_arguments_without_gpu():
    from paper_2109_08003_b200 import _capi
    st = _capi.lib.fnmt_linear(None, 0, 1, None, 0, None, None, 0, 1, 1, 1, 1, 0, None, 0, None)
    assert st == _capi.FNMT_E_INVALID
    assert b"fnmt_linear" in _capi.lib.fnmt_last_error()
    budgets = np.zeros(3, np.int32)
    lens = np.array([0, 10, 10_000], np.int32)
    total = _capi.lib.fnmt_budgets(lens.ctypes.data, 3, 1.5, 5, 64, budgets.ctypes.data)
    # search.py:49-51: 0 -> max(1, min(64, 5)) is only used for live rows; empty rows get 0
    assert list(budgets) == [0, 20, 64] and total == 84


# --- construction -------------------------------------------------------------

def test_random_model_bit_identical_to_oracle_and_reference(golden):
    g = golden("small_models")
    for tag in ("tiny", "tiny_unshared", "d64_h8_dec6"):
        c = [int(x) for x in g[f"{tag}__config"]]
        cfg = S.ModelConfig(*c[:9], norm_variant="l1" if c[9] else "l2",
                            shared_embeddings=bool(c[10]))
        w = S.random_model(cfg, int(g[f"{tag}__seed"]))
        assert sha(w.src_embed) == str(g[f"{tag}__src_embed_sha"])
        assert sha(w.enc_layers[0].attn.q.weight) == str(g[f"{tag}__enc0_q_sha"])
        assert S.count_params(cfg) == int(g[f"{tag}__count_params"])
        a = O.arch_of(cfg)
        p = O.make_params(a, int(g[f"{tag}__seed"]))
        named = dict(S.iter_named_tensors(cfg, w))
        for name, arr in named.items():
            want = p[name]
            assert np.array_equal(arr, want), name


def test_student_counts_and_positions(golden):
    g = golden("students")
    cfg = S.ModelConfig(6, 1, 512, 1, 1, 2048, 2048, 32772, 1024)
    assert S.count_params(cfg) == int(g["student_6_1_1_count"]) == 39_930_372
    k = golden("known_answers")
    assert sha(S.sinusoid_positions(1024, 512)) == str(k["positions_1024x512_sha"])
    assert sha(S.sinusoid_positions(1024, 768)) == str(k["positions_1024x768_sha"])


def test_config_validation():
    with pytest.raises(ValueError):
        S.ModelConfig(2, 1, 10, 3, 1, 32, 16, 48, 64)
    with pytest.raises(ValueError):
        S.ModelConfig(2, 0, 16, 2, 1, 32, 16, 48, 64)
    with pytest.raises(ValueError):
        S.ModelConfig(2, 1, 16, 2, 1, 32, 16, 48, 64, norm_variant="l3")


# --- batching -------------------------------------------------------------------

def test_batching_matches_reference_golden(golden):
    g = golden("batching")
    for i in range(6):
        lengths = [int(x) for x in g[f"c{i}_lengths"]]
        sb, wb = (int(x) for x in g[f"c{i}_caps"])
        plan = B.plan_batches(lengths, B.DecodeLimits(sbatch=sb, wbatch=wb))
        assert list(plan.permutation) == [int(x) for x in g[f"c{i}_perm"]]
        assert [len(b.indices) for b in plan.batches] == [int(x) for x in g[f"c{i}_sizes"]]
        assert [b.oversize for b in plan.batches] == [bool(x) for x in g[f"c{i}_oversize"]]
        assert B.restore_order(list(plan.permutation), plan) == list(range(len(lengths)))


@pytest.mark.parametrize("seed", range(20))
def test_batching_fuzz_against_oracle(seed):
    rng = np.random.default_rng(seed)
    lengths = [int(x) for x in rng.integers(1, 300, size=int(rng.integers(0, 80)))]
    sb, wb = int(rng.integers(1, 20)), int(rng.integers(8, 900))
    plan = B.plan_batches(lengths, B.DecodeLimits(sbatch=sb, wbatch=wb))
    batches, perm = O.plan(lengths, sb, wb)
    assert list(plan.permutation) == perm
    assert [(list(b.indices), b.max_len, b.oversize) for b in plan.batches] == \
        [(list(b[0]), b[1], b[2]) for b in batches]
    cfg = S.ModelConfig(2, 1, 16, 2, 1, 32, 16, 48, 64)
    assert B.estimate_peak_memory(plan, cfg, 40) == O.peak_bytes(batches, O.arch_of(cfg), 40)


def test_native_planner_matches_reference_golden(golden):
    """The planner the product runs (engine.cu plan_batches via the C ABI)
    against the reference's recorded plans (batching.py:100-109)."""
    from paper_2109_08003_b200.engine import native_plan
    g = golden("batching")
    for i in range(6):
        lengths = [int(x) for x in g[f"c{i}_lengths"]]
        sb, wb = (int(x) for x in g[f"c{i}_caps"])
        perm, batches = native_plan(lengths, sb, wb)
        assert perm == [int(x) for x in g[f"c{i}_perm"]]
        assert [len(b[0]) for b in batches] == [int(x) for x in g[f"c{i}_sizes"]]
        assert [b[1] for b in batches] == [int(x) for x in g[f"c{i}_maxlen"]]
        assert [b[2] for b in batches] == [bool(x) for x in g[f"c{i}_oversize"]]


@pytest.mark.parametrize("seed", range(20))
def test_native_planner_fuzz_against_oracle(seed):
    from paper_2109_08003_b200.engine import native_plan
    rng = np.random.default_rng(100 + seed)
    lengths = [int(x) for x in rng.integers(1, 300, size=int(rng.integers(0, 200)))]
    sb, wb = int(rng.integers(1, 40)), int(rng.integers(8, 2000))
    perm, batches = native_plan(lengths, sb, wb)
    want, wperm = O.plan(lengths, sb, wb)
    assert perm == wperm
    assert batches == [(list(b[0]), b[1], b[2]) for b in want]


def test_native_planner_corpus_scale():
    """At the bench's caps over a 65 536-sentence newstest-shaped chunk the
    native plan equals the Python restatement batch for batch."""
    from paper_2109_08003_b200.engine import native_plan
    from paper_2109_08003_b200.synthetic import newstest_lengths
    lengths = newstest_lengths(65536)
    perm, batches = native_plan(lengths, 3072, 64000)
    plan = B.plan_batches([int(x) for x in lengths], B.DecodeLimits(sbatch=3072, wbatch=64000))
    assert perm == list(plan.permutation)
    assert [(b[0], b[1], b[2]) for b in batches] == \
        [(list(b.indices), b.max_len, b.oversize) for b in plan.batches]


def test_restore_order_integrity():
    plan = B.plan_batches([4, 4], B.DecodeLimits())
    with pytest.raises(B.IntegrityError):
        B.restore_order(["x"], plan)


# --- search semantics on toy models (reference tests/test_search.py idioms) ------

class ToyCache:
    def __init__(self, prefixes):
        self.prefixes = prefixes
        self.step = 0

    def select(self, rows):
        c = ToyCache([list(self.prefixes[r]) for r in rows])
        c.step = self.step
        return c


class Toy:
    def __init__(self, table, vocab, max_positions=16):
        self.table = {k: np.asarray(v, np.float32) for k, v in table.items()}
        self.vocab = vocab
        self.max_positions = max_positions

    def init_cache(self, enc):
        return ToyCache([[] for _ in range(len(enc.pad_mask))])

    def step(self, cache, prev):
        if cache.step > 0:
            for row, tok in zip(cache.prefixes, prev):
                row.append(int(tok))
        cache.step += 1
        out = np.full((len(cache.prefixes), self.vocab), -1e9, np.float32)
        for b, row in enumerate(cache.prefixes):
            if tuple(row) in self.table:
                out[b] = self.table[tuple(row)]
            else:
                out[b, 3] = 0.0
        return out


def toy_enc(n, s=4):
    return SimpleNamespace(pad_mask=np.ones((n, s), bool))


def beam_toy():
    neg = -1e9

    def row(d):
        r = [neg] * 7
        for t, p in d.items():
            r[t] = math.log(p)
        return r
    return Toy({(): row({4: 0.6, 5: 0.4}), (4,): row({6: 0.55, 3: 0.45}),
                (5,): row({3: 0.9, 4: 0.05, 6: 0.05}), (4, 6): row({3: 1.0})}, 7)


def test_search_semantics_on_toys():
    from paper_2109_08003_b200.search import SearchConfig, beam_translate, greedy_translate, max_out_length
    cfg = SearchConfig(bos_id=2, eos_id=3, pad_id=0)
    assert max_out_length(0, cfg, 512) == 5 and max_out_length(10, cfg, 512) == 20
    assert max_out_length(10_000, cfg, 64) == 64
    assert greedy_translate(Toy({}, 7), toy_enc(3), cfg) == [[], [], []]
    assert greedy_translate(beam_toy(), toy_enc(1), cfg) == [[4, 6]]
    assert greedy_translate(Toy({}, 7), toy_enc(0), cfg) == []
    b1 = SearchConfig(bos_id=2, eos_id=3, pad_id=0, beam_size=1)
    b2 = SearchConfig(bos_id=2, eos_id=3, pad_id=0, beam_size=2)
    assert beam_translate(beam_toy(), toy_enc(1), b1) == [[4, 6]]
    assert beam_translate(beam_toy(), toy_enc(1), b2) == [[5]]
    tie = Toy({(): [-1e9] * 4 + [math.log(0.5)] * 2}, 6)
    assert greedy_translate(tie, toy_enc(1), cfg)[0][0] == 4
    assert beam_translate(tie, toy_enc(1), b1)[0][0] == 4


def test_search_matches_oracle_on_small_models(golden):
    """The host search loop driven by the oracle's decoder reproduces the
    reference's recorded greedy / beam outputs (pins search.py semantics)."""
    from paper_2109_08003_b200.search import SearchConfig, beam_translate, greedy_translate
    g = golden("small_models")

    class OracleModel:
        def __init__(self, a, p):
            self.a, self.p, self.max_positions = a, p, a.max_positions

        def init_cache(self, enc):
            c = O.start_cache(self.a, self.p, enc.states, enc.pad_mask)

            class Cache:
                pass
            box = Cache()
            box.c = c
            box.select = lambda rows: _wrap(O.pick_rows(box.c, rows))
            return box

        def step(self, cache, prev):
            return O.decoder_step(self.a, self.p, cache.c, prev)

    def _wrap(c):
        class Cache:
            pass
        box = Cache()
        box.c = c
        box.select = lambda rows: _wrap(O.pick_rows(box.c, rows))
        return box

    for tag in ("tiny", "tiny_dec2_h2", "d64_h8_dec6"):
        c = [int(x) for x in g[f"{tag}__config"]]
        a = O.Arch(*c[:9], norm_variant="l1" if c[9] else "l2", shared_embeddings=bool(c[10]))
        p = O.make_params(a, int(g[f"{tag}__seed"]))
        tok, valid = g[f"{tag}__tokens"], g[f"{tag}__valid"]
        enc = SimpleNamespace(states=O.encoder(a, p, tok, valid), pad_mask=valid)
        m = OracleModel(a, p)
        split = lambda ids, lens: [list(map(int, ids[o:o + n])) for o, n in
                                   zip(np.concatenate([[0], np.cumsum(lens)[:-1]]), lens)]
        want = split(g[f"{tag}__greedy_ids"], g[f"{tag}__greedy_lens"])
        assert greedy_translate(m, enc, SearchConfig(2, 3, 0)) == want
        for k in (2, 4):
            want = split(g[f"{tag}__beam{k}_ids"], g[f"{tag}__beam{k}_lens"])
            assert beam_translate(m, enc, SearchConfig(2, 3, 0, beam_size=k)) == want


def test_device_workspace_estimate_pinned():
    """batching.estimate_device_bytes against the workspace the engine
    allocated on a B200 (tests/test_gpu_memory.py, profiles/r02/
    gpu_tests_summary.txt): the folded single-head, multi-head and fp32
    layouts at the paper's caps and at small caps."""
    from paper_2109_08003_b200 import store as S
    from paper_2109_08003_b200.batching import estimate_device_bytes
    measured = {(1, 2, 3072, 64000): 1265375252, (1, 2, 128, 2048): 41287316,
                (8, 2, 3072, 64000): 1262520340, (8, 2, 128, 2048): 41193108,
                (1, 4, 3072, 64000): 2111866900, (1, 4, 128, 2048): 68980372}
    for (heads, es, sb, wb), want in measured.items():
        cfg = S.ModelConfig(6, 1, 512, heads, heads, 2048, 2048, 32772, 1024)
        assert estimate_device_bytes(cfg, sb, wb, dtype_bytes=es) == want, (heads, es, sb, wb)
