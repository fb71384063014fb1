"""GPU kernel parity through the C ABI (sm_100a).

GEMMs are checked against a plain PyTorch fp32 matmul of the same (rounded)
operands; row kernels and attention against the CPU oracle."""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import nmt_oracle as O  # noqa: E402
from paper_2109_08003_b200 import _capi  # noqa: E402
from paper_2109_08003_b200._capi import check, lib, ptr  # noqa: E402

DEV = torch.device("cuda", 0)
TDT = {_capi.F16: torch.float16, _capi.BF16: torch.bfloat16, _capi.F32: torch.float32}


def stream():
    return torch.cuda.current_stream().cuda_stream


def linear(A, W, bias, dt, out_dt=_capi.F32, relu=0, resid=None):
    M, K = A.shape
    N = W.shape[0]
    C = torch.empty((M, N), dtype=TDT[out_dt], device=DEV)
    check(lib.fnmt_linear(ptr(A), K, dt, ptr(W), K, ptr(bias), ptr(C), N, out_dt, M, N, K, relu,
                          ptr(resid), N if resid is not None else 0, stream()), "linear")
    torch.cuda.synchronize()
    return C


SHAPES = [(1, 16, 16), (5, 48, 16), (77, 130, 64), (128, 128, 512), (300, 512, 512),
          (257, 1536, 512), (1000, 2048, 512), (999, 512, 2048), (64, 32772, 512),
          (3, 96, 768), (130, 768, 3072), (8200, 1536, 512), (8320, 512, 2048)]


@pytest.mark.parametrize("dt", [_capi.F16, _capi.BF16])
@pytest.mark.parametrize("M,N,K", SHAPES)
def test_tcgen05_gemm_matches_fp32_reference(dt, M, N, K):
    g = torch.Generator(device="cpu").manual_seed(M * 7 + N * 3 + K)
    A = torch.randn(M, K, generator=g).to(DEV, TDT[dt])
    W = (torch.randn(N, K, generator=g) / math.sqrt(K)).to(DEV, TDT[dt])
    bias = (torch.randn(N, generator=g) * 0.1).to(DEV)
    ref = A.float() @ W.float().T + bias
    got = linear(A, W, bias, dt)
    err = (got - ref).abs().max().item()
    assert err <= 2e-3 * max(1.0, ref.abs().max().item()), err
    # fused ReLU + 16-bit store
    got16 = linear(A, W, bias, dt, out_dt=dt, relu=1)
    want16 = torch.relu(ref).to(TDT[dt]).float()
    assert (got16.float() - want16).abs().max().item() <= 2e-2 * max(1.0, want16.abs().max().item())


def test_tcgen05_gemm_batch_invariance():
    """A row's result must not depend on M (fixed k order, no split-K)."""
    g = torch.Generator(device="cpu").manual_seed(5)
    A = torch.randn(700, 512, generator=g).to(DEV, torch.float16)
    W = (torch.randn(1536, 512, generator=g) / 22.6).to(DEV, torch.float16)
    bias = torch.zeros(1536, device=DEV)
    full = linear(A, W, bias, _capi.F16)
    for lo, hi in [(0, 1), (3, 130), (611, 700)]:
        part = linear(A[lo:hi].contiguous(), W, bias, _capi.F16)
        assert torch.equal(part, full[lo:hi])


@pytest.mark.parametrize("M,N,K", [(1, 16, 16), (77, 130, 64), (300, 512, 512), (33, 1000, 2048)])
def test_simt_fp32_gemm(M, N, K):
    rng = np.random.default_rng(M + N + K)
    a = rng.standard_normal((M, K)).astype(np.float32)
    w = rng.standard_normal((K, N)).astype(np.float32) / np.float32(math.sqrt(K))
    b = rng.standard_normal(N).astype(np.float32)
    A = torch.from_numpy(a).to(DEV)
    Wt = torch.from_numpy(np.ascontiguousarray(w.T)).to(DEV)
    got = linear(A, Wt, torch.from_numpy(b).to(DEV), _capi.F32).cpu().numpy()
    want = O.mm(a, w) + b
    assert np.abs(got - want).max() <= 1e-4 * max(1.0, np.abs(want).max())


@pytest.mark.parametrize("dt", [_capi.F16, _capi.F32])
@pytest.mark.parametrize("M", [200, 1100])
def test_fused_vocab_argmax_lowest_id_on_ties(dt, M):
    g = torch.Generator(device="cpu").manual_seed(11)
    N, K = 32772, 512
    A = torch.randn(M, K, generator=g).to(DEV, TDT[dt])
    W = (torch.randn(N, K, generator=g) / 22.6).to(DEV, TDT[dt])
    W[7] = W[5]            # exact duplicate column -> tie between ids 5 and 7
    W[32771] = W[5]
    bias = torch.zeros(N, device=DEV)
    bias[5] = 100.0
    bias[7] = 100.0
    bias[32771] = 100.0
    keys = torch.zeros(M, dtype=torch.int64, device=DEV)
    idx = torch.empty(M, dtype=torch.int32, device=DEV)
    check(lib.fnmt_linear_argmax(ptr(A), K, dt, ptr(W), K, ptr(bias), M, N, K, ptr(keys),
                                 ptr(idx), stream()), "argmax")
    torch.cuda.synchronize()
    assert (idx == 5).all()
    bias[5] = bias[7] = bias[32771] = 0.0
    check(lib.fnmt_linear_argmax(ptr(A), K, dt, ptr(W), K, ptr(bias), M, N, K, ptr(keys),
                                 ptr(idx), stream()), "argmax")
    logits = linear(A, W, bias, dt)
    torch.cuda.synchronize()
    ref = logits.argmax(dim=1).to(torch.int32)
    assert (idx == ref).float().mean().item() == 1.0


@pytest.mark.parametrize("dt", [_capi.F16, _capi.BF16])
@pytest.mark.parametrize("M,N,K", [(3072, 32772, 512), (129, 1000, 64), (300, 4100, 448),
                                   (1500, 9000, 576)])
def test_fused_vocab_argmax_shapes(dt, M, N, K):
    """The fused vocab argmax (BN = 256 tiles, N tails, K = 64..576) is the
    argmax of the same GEMM's fp32 logits."""
    g = torch.Generator(device="cpu").manual_seed(M + N + K)
    A = torch.randn(M, K, generator=g).to(DEV, TDT[dt])
    W = (torch.randn(N, K, generator=g) / K ** 0.5).to(DEV, TDT[dt])
    bias = (torch.randn(N, generator=g) * 0.1).to(DEV)
    keys = torch.zeros(M, dtype=torch.int64, device=DEV)
    idx = torch.empty(M, dtype=torch.int32, device=DEV)
    check(lib.fnmt_linear_argmax(ptr(A), K, dt, ptr(W), K, ptr(bias), M, N, K, ptr(keys),
                                 ptr(idx), stream()), "argmax")
    logits = linear(A, W, bias, dt)
    torch.cuda.synchronize()
    ref = logits.argmax(dim=1).to(torch.int32)
    assert (idx == ref).all()


@pytest.mark.parametrize("variant", ["l2", "l1"])
@pytest.mark.parametrize("d", [16, 64, 512, 768])
def test_add_norm_matches_oracle(variant, d):
    rng = np.random.default_rng(d)
    x = (rng.standard_normal((37, d)) * 3 + 1).astype(np.float32)
    y = rng.standard_normal((37, d)).astype(np.float32)
    x[3] = 5.0
    y[3] = 0.0                          # constant row -> exactly bias
    g = rng.standard_normal(d).astype(np.float32)
    b = rng.standard_normal(d).astype(np.float32)
    X, Y, G, Bb = (torch.from_numpy(v).to(DEV) for v in (x, y, g, b))
    out = torch.empty_like(X)
    out16 = torch.empty(X.shape, dtype=torch.float16, device=DEV)
    check(lib.fnmt_add_norm(ptr(X), ptr(Y), ptr(G), ptr(Bb), int(variant == "l1"), ptr(out),
                            ptr(out16), _capi.F16, 37, d, stream()), "norm")
    torch.cuda.synchronize()
    want = O.norm_rows(variant, x + y, g, b)
    got = out.cpu().numpy()
    assert np.abs(got - want).max() <= 1e-5 * max(1.0, np.abs(want).max())
    assert np.array_equal(got[3], b)
    assert np.allclose(out16.float().cpu().numpy(), got, atol=1e-2, rtol=1e-3)


def test_embed_matches_oracle():
    rng = np.random.default_rng(0)
    V, d = 100, 64
    table = rng.standard_normal((V, d)).astype(np.float32)
    pos = O.position_table(32, d)
    ids = rng.integers(0, V, size=50).astype(np.int32)
    pids = rng.integers(0, 32, size=50).astype(np.int32)
    T, P, I, PI = (torch.from_numpy(v).to(DEV) for v in (table, pos, ids, pids))
    out = torch.empty((50, d), device=DEV)
    check(lib.fnmt_embed(ptr(I), ptr(PI), ptr(T), ptr(P), float(np.float32(math.sqrt(d))),
                         ptr(out), None, _capi.F32, 50, d, stream()), "embed")
    torch.cuda.synchronize()
    want = table[ids] * np.float32(math.sqrt(d)) + pos[pids]
    assert np.array_equal(out.cpu().numpy(), want)


@pytest.mark.parametrize("heads,d", [(1, 16), (2, 16), (8, 32), (1, 512), (8, 512), (8, 768)])
def test_varlen_attention_matches_oracle(heads, d):
    rng = np.random.default_rng(heads * 100 + d)
    lens = [7, 1, 23, 40]
    s = max(lens)
    b = len(lens)
    q = rng.standard_normal((b, s, d)).astype(np.float32)
    k = rng.standard_normal((b, s, d)).astype(np.float32)
    v = rng.standard_normal((b, s, d)).astype(np.float32)
    valid = np.arange(s)[None, :] < np.array(lens)[:, None]
    want = O.mha(q, k, v, O.key_mask(valid), heads)
    Q, K_, V_ = (torch.from_numpy(a.reshape(b * s, d)).to(DEV) for a in (q, k, v))
    out = torch.zeros((b * s, d), device=DEV)
    start = torch.arange(b, dtype=torch.int32, device=DEV) * s
    qlen = torch.full((b,), s, dtype=torch.int32, device=DEV)
    klen = torch.tensor(lens, dtype=torch.int32, device=DEV)
    check(lib.fnmt_attention(ptr(Q), d, ptr(K_), ptr(V_), d, ptr(out), d, _capi.F32, heads,
                             d // heads, ptr(start), ptr(qlen), ptr(start), ptr(klen), s, b, s, s,
                             stream()), "attention")
    torch.cuda.synchronize()
    got = out.cpu().numpy().reshape(b, s, d)
    assert np.abs(got - want).max() <= 2e-5


def test_attention_all_masked_row_follows_reference():
    """A row with no real key attends uniformly-ish over padded keys with the
    -1e9 offset (model.py:243-245) instead of producing NaN."""
    rng = np.random.default_rng(3)
    b, s, d = 2, 5, 16
    q = rng.standard_normal((b, s, d)).astype(np.float32)
    k = rng.standard_normal((b, s, d)).astype(np.float32)
    v = rng.standard_normal((b, s, d)).astype(np.float32)
    valid = np.array([[1, 1, 1, 0, 0], [0, 0, 0, 0, 0]], bool)
    want = O.mha(q, k, v, O.key_mask(valid), 2)
    Q, K_, V_ = (torch.from_numpy(a.reshape(b * s, d)).to(DEV) for a in (q, k, v))
    out = torch.zeros((b * s, d), device=DEV)
    start = torch.arange(b, dtype=torch.int32, device=DEV) * s
    qlen = torch.full((b,), s, dtype=torch.int32, device=DEV)
    klen = torch.tensor([3, 0], dtype=torch.int32, device=DEV)
    check(lib.fnmt_attention(ptr(Q), d, ptr(K_), ptr(V_), d, ptr(out), d, _capi.F32, 2, 8,
                             ptr(start), ptr(qlen), ptr(start), ptr(klen), s, b, s, s, stream()),
          "attention")
    torch.cuda.synchronize()
    assert np.abs(out.cpu().numpy().reshape(b, s, d) - want).max() <= 1e-5


@pytest.mark.parametrize("heads,d,lens", [(1, 512, [7, 1, 23, 40]), (8, 512, [24, 3, 65, 17]),
                                          (8, 768, [9, 31]), (2, 64, [200, 130, 5]),
                                          (1, 64, [300, 12]), (4, 64, [0, 6])])
def test_varlen_attention_f16_tensor_core(heads, d, lens):
    """fp16 storage: the mma.sync encoder attention (<= 256 keys) and the SIMT
    fallback (longer) against the fp32 oracle on fp16-rounded inputs; a
    zero-length key set exercises the all-masked -1e9 rule."""
    rng = np.random.default_rng(heads * 1000 + d + len(lens))
    b, s = len(lens), max(max(lens), 1)
    q, k, v = (rng.standard_normal((b, s, d)).astype(np.float16).astype(np.float32)
               for _ in range(3))
    valid = np.arange(s)[None, :] < np.array(lens)[:, None]
    want = O.mha(q, k, v, O.key_mask(valid), heads)
    Q, K_, V_ = (torch.from_numpy(a.reshape(b * s, d)).half().to(DEV) for a in (q, k, v))
    out = torch.zeros((b * s, d), device=DEV, dtype=torch.float16)
    start = torch.arange(b, dtype=torch.int32, device=DEV) * s
    qlen = torch.full((b,), s, dtype=torch.int32, device=DEV)
    klen = torch.tensor(lens, dtype=torch.int32, device=DEV)
    check(lib.fnmt_attention(ptr(Q), d, ptr(K_), ptr(V_), d, ptr(out), d, _capi.F16, heads,
                             d // heads, ptr(start), ptr(qlen), ptr(start), ptr(klen), s, b, s, s,
                             stream()), "attention")
    torch.cuda.synchronize()
    got = out.float().cpu().numpy().reshape(b, s, d)
    assert np.abs(got - want).max() <= 1e-2 * max(1.0, np.abs(want).max())


@pytest.mark.parametrize("dt", ["f16", "bf16"])
@pytest.mark.parametrize("M,N,K,l1", [(3, 512, 512, 0), (300, 512, 2048, 0), (1000, 512, 512, 1),
                                      (130, 768, 768, 0), (77, 256, 64, 1), (50, 96, 64, 0)])
def test_linear_add_norm_fused(dt, M, N, K, l1):
    """x = norm(x + A W^T + b) (GEMM adding into x in its epilogue, then the
    row norm) against the fp32 oracle on storage-rounded operands."""
    rng = np.random.default_rng(M + N + K)
    tdt = torch.float16 if dt == "f16" else torch.bfloat16
    A = torch.from_numpy(rng.standard_normal((M, K)).astype(np.float32)).to(tdt)
    W = torch.from_numpy((rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32)).to(tdt)
    b = rng.standard_normal(N).astype(np.float32) * 0.1
    x = rng.standard_normal((M, N)).astype(np.float32)
    g = (1 + 0.1 * rng.standard_normal(N)).astype(np.float32)
    be = (0.1 * rng.standard_normal(N)).astype(np.float32)
    y = A.float().numpy() @ W.float().numpy().T + b
    want = O.norm_rows("l1" if l1 else "l2", x + y, g, be)
    Ad, Wd = A.to(DEV), W.to(DEV)
    X = torch.from_numpy(x).to(DEV)
    Xa = torch.empty((M, N), dtype=tdt, device=DEV)
    B, G, Be = (torch.from_numpy(v).to(DEV) for v in (b, g, be))
    check(lib.fnmt_linear_add_norm(ptr(Ad), K, _capi.DTYPES[dt], ptr(Wd), K, ptr(B), ptr(X),
                                   ptr(Xa), ptr(G), ptr(Be), l1, M, N, K, stream()), "add_norm")
    torch.cuda.synchronize()
    got = X.cpu().numpy()
    assert np.abs(got - want).max() <= 2e-3 * max(1.0, np.abs(want).max())
    assert np.allclose(Xa.float().cpu().numpy(), got, atol=3e-2, rtol=1e-2)
