"""Subprocess body of test_cta_pair_gemm (FNMT_GEMM_PAIR=1 must be set before
the library's first GEMM): the cta_group::2 GEMM against a PyTorch fp32
matmul of the same operands, store and fused-argmax epilogues."""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2109_08003_b200 import _capi  # noqa: E402
from paper_2109_08003_b200._capi import check, lib, ptr  # noqa: E402

DEV = torch.device("cuda", 0)
TDT = {_capi.F16: torch.float16, _capi.BF16: torch.bfloat16}


def main():
    s = torch.cuda.current_stream().cuda_stream
    for dt in (_capi.F16, _capi.BF16):
        for M, N, K in [(20000, 512, 512), (4096, 4096, 512), (3001, 2048, 2048),
                        (19000, 1536, 512), (256 * 75, 256, 64)]:
            g = torch.Generator(device="cpu").manual_seed(M + N + K)
            A = torch.randn(M, K, generator=g).to(DEV, TDT[dt])
            W = (torch.randn(N, K, generator=g) / math.sqrt(K)).to(DEV, TDT[dt])
            b = (torch.randn(N, generator=g) * 0.1).to(DEV)
            C = torch.empty((M, N), device=DEV)
            check(lib.fnmt_linear(ptr(A), K, dt, ptr(W), K, ptr(b), ptr(C), N, _capi.F32, M, N, K,
                                  0, None, 0, s), "linear")
            torch.cuda.synchronize()
            ref = A.float() @ W.float().T + b
            err = (C - ref).abs().max().item()
            assert err <= 2e-3 * max(1.0, ref.abs().max().item()), (dt, M, N, K, err)
        # fused vocab argmax: M rows x 32772
        M, N, K = 3000, 32772, 512
        g = torch.Generator(device="cpu").manual_seed(5)
        A = torch.randn(M, K, generator=g).to(DEV, TDT[dt])
        W = (torch.randn(N, K, generator=g) / math.sqrt(K)).to(DEV, TDT[dt])
        b = (torch.randn(N, generator=g) * 0.1).to(DEV)
        keys = torch.zeros(M, dtype=torch.int64, device=DEV)
        idx = torch.empty(M, dtype=torch.int32, device=DEV)
        check(lib.fnmt_linear_argmax(ptr(A), K, dt, ptr(W), K, ptr(b), M, N, K, ptr(keys),
                                     ptr(idx), s), "argmax")
        torch.cuda.synchronize()
        logits = A.float() @ W.float().T + b
        top2 = logits.topk(2, dim=1).values
        got = idx.long()
        ok = (got == logits.argmax(dim=1)) | ((top2[:, 0] - top2[:, 1]) < 1e-3)
        assert bool(ok.all()), int((~ok).sum())
    print("pair gemm ok")


if __name__ == "__main__":
    main()
