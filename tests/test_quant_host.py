"""int8 scheme on the host (CPU): the oracle restatement and the product's
load-time weight quantization, bit-exact against the reference fixtures."""

import hashlib
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import quant_oracle as QO
from paper_2109_08003_b200 import quant8 as Q

sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "oracle"))
from make_golden_quant import CASES, case_inputs  # noqa: E402  (input recipe only)


def sha(x):
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def gq(golden):
    return golden("quant8")


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_oracle_matches_reference(gq, case):
    tag = case[0]
    a, w = case_inputs(*case)
    assert sha(a) == str(gq[f"{tag}__a_sha"]) and sha(w) == str(gq[f"{tag}__w_sha"])
    q, s, z = QO.quantize_weights(w)
    assert sha(q) == str(gq[f"{tag}__wq_sha"])
    assert sha(s) == str(gq[f"{tag}__wscale_sha"]) and sha(z) == str(gq[f"{tag}__wzp_sha"])
    aq, asc, azp = QO.quantize_activations(a)
    assert sha(aq) == str(gq[f"{tag}__aq_sha"])
    assert asc == float(gq[f"{tag}__ascale"]) and azp == float(gq[f"{tag}__azp"])
    c = QO.qgemm(aq, asc, azp, q, s, z)
    assert sha(c) == str(gq[f"{tag}__c_sha"])


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_product_weight_quantization_matches_reference(gq, case):
    tag = case[0]
    _, w = case_inputs(*case)
    qm = Q.quantize_weights(w)
    assert sha(qm.q) == str(gq[f"{tag}__wq_sha"])
    assert sha(qm.col_scale) == str(gq[f"{tag}__wscale_sha"])
    assert sha(qm.col_zeropoint) == str(gq[f"{tag}__wzp_sha"])


def test_device_operands_layout():
    rng = np.random.default_rng(0)
    w = rng.standard_normal((40, 24)).astype(np.float32)
    qm = Q.quantize_weights(w)
    wt, sc, zp, cs = Q.device_operands(qm)
    assert wt.shape == (24, 48) and wt.dtype == np.int8
    assert np.array_equal(wt[:, :40], qm.q.T) and not wt[:, 40:].any()
    assert np.array_equal(cs, qm.q.astype(np.int64).sum(0))


def test_small_case_full_arrays(gq):
    a, w = gq["small__a"], gq["small__w"]
    q, s, z = QO.quantize_weights(w)
    assert np.array_equal(q, gq["small__wq"])
    assert s[3] == 1.0                         # degenerate column
    aq, asc, azp = QO.quantize_activations(gq["k_tiny__a"])
    assert asc == 1.0 and np.all(aq == 255)    # constant activations clamp to 255
