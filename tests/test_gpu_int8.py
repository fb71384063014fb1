"""int8 path on the GPU: ``fnmt_qgemm`` (tcgen05 kind::i8) bit-exact against
the reference's qgemm (tests/golden/quant8.npz via the pinned oracle), and the
int8 engine end to end against the reference's int8 model."""

import ctypes as C
import sys
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import quant_oracle as QO  # noqa: E402
from paper_2109_08003_b200 import quant8 as Q  # noqa: E402
from paper_2109_08003_b200 import store as S  # noqa: E402
from paper_2109_08003_b200._capi import check, lib  # noqa: E402
from paper_2109_08003_b200.model import GpuTranslationModel  # noqa: E402
from paper_2109_08003_b200.search import SearchConfig, greedy_translate  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "oracle"))
from make_golden_quant import CASES, case_inputs  # noqa: E402

DEV = torch.device("cuda:0")


def qgemm_gpu(a, w, bias=None, relu=0, lda_pad=0):
    m, k = a.shape
    qm = Q.quantize_weights(w)
    wt, sc, zp, cs = Q.device_operands(qm)
    n = wt.shape[0]
    A = torch.zeros((m, k + lda_pad), dtype=torch.float32, device=DEV)
    A[:, :k] = torch.from_numpy(a).to(DEV)
    d = {x: torch.from_numpy(v).to(DEV) for x, v in dict(wt=wt, sc=sc, zp=zp, cs=cs).items()}
    b = torch.from_numpy(np.asarray(bias, np.float32)).to(DEV) if bias is not None else None
    Cm = torch.empty((m, n), dtype=torch.float32, device=DEV)
    nb = lib.fnmt_qgemm_workspace(m, k)
    ws = torch.empty(nb, dtype=torch.uint8, device=DEV)
    check(lib.fnmt_qgemm(A.data_ptr(), k + lda_pad, d["wt"].data_ptr(), d["sc"].data_ptr(),
                         d["zp"].data_ptr(), d["cs"].data_ptr(), b.data_ptr() if b is not None
                         else None, Cm.data_ptr(), n, m, n, k, relu, ws.data_ptr(), nb, None),
          "qgemm")
    torch.cuda.synchronize()
    return Cm.cpu().numpy()


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_qgemm_bit_exact(case):
    a, w = case_inputs(*case)
    q, s, z = QO.quantize_weights(w)
    aq, asc, azp = QO.quantize_activations(a)
    want = QO.qgemm(aq, asc, azp, q, s, z)
    got = qgemm_gpu(a, w)
    assert np.array_equal(got, want), np.abs(got - want).max()


def test_qgemm_bias_relu_and_strided_input():
    a, w = case_inputs("k_ragged", 33, 40, 72, 2)
    bias = np.random.default_rng(3).standard_normal(72).astype(np.float32)
    want = np.maximum(QO.linear(a, w, bias), np.float32(0))
    assert np.array_equal(qgemm_gpu(a, w, bias, relu=1, lda_pad=8), want)


def test_qgemm_batch_shape_independent():
    # same activations matrix split differently => the integer core is exact
    # per element; only the activation scale (whole-matrix min / max) couples rows
    a, w = case_inputs("proj_512", 300, 512, 512, 4)
    full = qgemm_gpu(a, w)
    q, s, z = QO.quantize_weights(w)
    aq, asc, azp = QO.quantize_activations(a)
    assert np.array_equal(full, QO.qgemm(aq, asc, azp, q, s, z))


def test_int8_engine_greedy_matches_reference(golden):
    g = golden("int8_models")
    same = total = 0
    for tag in [str(t) for t in g["tags"]]:
        c = [int(x) for x in g[f"{tag}__config"]]
        cfg = S.ModelConfig(*c)
        w = S.random_model(cfg, int(g[f"{tag}__seed"]))
        m = GpuTranslationModel(cfg, w, dtype="int8")
        tok = g[f"{tag}__tokens"]
        got = greedy_translate(m, m.encode(tok, np.ones_like(tok, bool)), SearchConfig(2, 3, 0))
        lens, flat = g[f"{tag}__out_len"], g[f"{tag}__out_ids"]
        want, o = [], 0
        for L in lens:
            want.append([int(x) for x in flat[o:o + L]])
            o += int(L)
        same += sum(a == b for a, b in zip(got, want))
        total += len(want)
    # the per-GEMM activation quantization is a rounding step: an f32 ulp of
    # difference upstream can move one level; require >= 90% identical
    assert same >= 0.9 * total, (same, total)


def test_int8_translator_worker_invariance():
    from paper_2109_08003_b200.textpipe import synthetic_vocabulary
    from paper_2109_08003_b200.translator import RunConfig, Translator
    cfg = S.ModelConfig(2, 1, 32, 2, 1, 64, 32, 96, 96)
    t = Translator(cfg, S.random_model(cfg, 0), synthetic_vocabulary(96),
                   run=RunConfig(precision="int8", chunk_lines=6))
    lines = [" ".join(["a", "b", "c"][: 1 + i % 3]) + f" {i}" for i in range(30)]
    a = t.translate_lines(lines)
    assert t.with_run(workers=4).translate_lines(lines) == a
    assert len(a) == 30
