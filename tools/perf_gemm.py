"""GEMM shape microbenchmark for the tcgen05 kernel (fnmt_linear), warm L2,
launches captured in a CUDA graph and timed with CUDA events.

python tools/perf_gemm.py
"""

import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import sys

import torch

from paper_2109_08003_b200 import _capi
from paper_2109_08003_b200._capi import check, lib, ptr

SHAPES = [  # (M, N, K, note)
    (600, 512, 512, "dec o-proj, long batch"),
    (600, 1536, 512, "dec qkv, long batch"),
    (600, 2048, 512, "dec ffn1, long batch"),
    (600, 512, 2048, "dec ffn2, long batch"),
    (2000, 512, 512, "dec o-proj"),
    (2000, 1536, 512, "dec qkv"),
    (2000, 2048, 512, "dec ffn1"),
    (2000, 512, 2048, "dec ffn2"),
    (3072, 512, 512, "dec o-proj, short batch"),
    (2000, 32772, 512, "vocab (store f32)"),
    (64000, 1536, 512, "enc qkv"),
    (64000, 2048, 512, "enc ffn1"),
    (64000, 512, 2048, "enc ffn2"),
]


def bench(M, N, K, reps=20, out_dtype=_capi.F16):
    dev = torch.device("cuda")
    A = torch.randn(M, K, device=dev).half()
    W = (torch.randn(N, K, device=dev) / K ** 0.5).half()
    b = torch.zeros(N, device=dev)
    C = torch.empty(M, N, device=dev, dtype=torch.float16 if out_dtype == _capi.F16 else torch.float32)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            check(lib.fnmt_linear(ptr(A), K, _capi.F16, ptr(W), K, ptr(b), ptr(C), N, out_dtype, M, N,
                                  K, 0, None, 0, s.cuda_stream), "linear")
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (5 * reps)
    return us, 2.0 * M * N * K / (us * 1e-6) / 1e12


DEC = [  # decoder step shapes of Student-6-1-1 (folded self: N = 2d + 8)
    (3072, 1032, 512, "dec fsk (folded self k~|v~|c)"),
    (3072, 1024, 512, "dec fsk without the c tail"),
    (3072, 1040, 512, "dec fsk, 16-col tail"),
    (3072, 2048, 512, "dec ffn1"),
    (3072, 512, 2048, "dec ffn2"),
    (1100, 1032, 512, "dec fsk, long batch"),
    (1100, 2048, 512, "dec ffn1, long batch"),
    (1100, 512, 2048, "dec ffn2, long batch"),
]


def main():
    shapes = DEC if "dec" in sys.argv[1:] else SHAPES
    for M, N, K, note in shapes:
        us, tf = bench(M, N, K, out_dtype=_capi.F32 if "f32" in note else _capi.F16)
        print(f"M={M:6d} N={N:6d} K={K:5d}  {us:8.2f} us  {tf:7.1f} TFLOP/s  {note}")
    sys.stdout.flush()


if __name__ == "__main__":
    main()
