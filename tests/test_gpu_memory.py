"""Device memory against the estimate (the reference's
analogue is tests/test_acceptance.py:350-391, tracemalloc vs
estimate_peak_memory): the engine's workspace at the paper's GPU caps equals
batching.estimate_device_bytes allocation for allocation, for the folded
single-head (Student-6-1-1) and the multi-head (Student-6-1-8) layouts."""

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2109_08003_b200 import store as S  # noqa: E402
from paper_2109_08003_b200.batching import estimate_device_bytes  # noqa: E402
from paper_2109_08003_b200.engine import Engine  # noqa: E402


@pytest.mark.parametrize("heads,dtype,es", [(1, "f16", 2), (8, "f16", 2), (1, "bf16", 2),
                                            (1, "f32", 4)])
def test_workspace_matches_estimate(heads, dtype, es):
    cfg = S.ModelConfig(6, 1, 512, heads, heads, 2048, 2048, 32772, 1024)
    eng = Engine(cfg, S.random_model(cfg, 0), dtype=dtype)
    weights = eng.device_bytes()
    for sb, wb in ((3072, 64000), (128, 2048)):
        e2 = Engine(cfg, S.random_model(cfg, 0), dtype=dtype) if (sb, wb) != (3072, 64000) else eng
        w0 = e2.device_bytes()
        e2.reserve(sb, wb)
        got = e2.device_bytes() - w0
        want = estimate_device_bytes(cfg, sb, wb, dtype_bytes=es)
        print(heads, dtype, sb, wb, "workspace", got, "estimate", want, "weights", weights)
        assert got == want
