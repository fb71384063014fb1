"""Error behaviour of the drop-in (reference tests/test_model.py and
tests/test_search.py contracts): LengthError for sources / decode positions
beyond max_positions (model.py:41, :274, :324), ValueError for token ids out
of range (model.py:254-258), and the C ABI's status codes behind them."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2109_08003_b200 import store as S  # noqa: E402
from paper_2109_08003_b200._capi import FnmtLengthError  # noqa: E402
from paper_2109_08003_b200.engine import Engine  # noqa: E402
from paper_2109_08003_b200.model import GpuTranslationModel, LengthError  # noqa: E402
from paper_2109_08003_b200.search import SearchConfig, greedy_translate  # noqa: E402

CFG = S.ModelConfig(2, 1, 32, 2, 1, 64, 32, 48, 16)


@pytest.fixture(scope="module")
def model():
    return GpuTranslationModel(CFG, S.random_model(CFG, 0), dtype="f16")


def test_encode_rejects_long_source(model):
    tok = np.full((1, 17), 5, np.int64)
    with pytest.raises(LengthError):
        model.encode(tok, np.ones_like(tok, bool))


def test_encode_rejects_bad_token_ids(model):
    for bad in (-1, 48, 10 ** 6):
        tok = np.array([[4, bad, 5]], np.int64)
        with pytest.raises(ValueError):
            model.encode(tok, np.ones_like(tok, bool))


def test_step_rejects_positions_past_max(model):
    tok = np.full((2, 3), 7, np.int64)
    enc = model.encode(tok, np.ones_like(tok, bool))
    cache = model.init_cache(enc)
    prev = np.full(2, 2, np.int64)
    for _ in range(CFG.max_positions):
        model.step(cache, prev)
    with pytest.raises(LengthError):
        model.step(cache, prev)
    with pytest.raises(ValueError):
        model.step(model.init_cache(enc), np.array([2, 99], np.int64))


def test_greedy_budget_caps_at_max_positions(model):
    """max_out_length = min(max_positions, ceil(1.5 S) + 5) (search.py:49-51):
    a 15-token source has budget min(16, 28) = 16 and never overruns."""
    tok = np.full((1, 15), 9, np.int64)
    out = greedy_translate(model, model.encode(tok, np.ones_like(tok, bool)),
                           SearchConfig(2, 3, 0))
    assert len(out[0]) <= CFG.max_positions


def test_engine_translate_length_and_id_errors():
    eng = Engine(CFG, S.random_model(CFG, 0), dtype="f16")
    ids = np.full(20, 5, np.int32)
    with pytest.raises(FnmtLengthError):
        eng.translate(ids, np.array([0, 20], np.int64))
    with pytest.raises(ValueError):
        eng.translate(np.array([4, 60, 5], np.int32), np.array([0, 3], np.int64))
    # the engine is still usable after a rejected call
    out, olen, off, _ = eng.translate(np.array([4, 6, 5], np.int32), np.array([0, 3], np.int64))
    assert olen[0] >= 1
