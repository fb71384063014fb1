"""add_norm_kernel microbenchmark (fnmt_add_norm): x32 + y32 -> LayerNorm ->
out32 + fp16 copy, d = 512, graph-captured launches, CUDA events.
Bytes per row: 4d (x) + 4d (y) + 4d (out32) + 2d (fp16).

Usage: python tools/perf_norm.py [rows ...]"""

import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2109_08003_b200 import _capi  # noqa: E402
from paper_2109_08003_b200._capi import check, lib, ptr  # noqa: E402

d = 512
for M in [int(a) for a in sys.argv[1:]] or [64000, 16000, 3072]:
    x = torch.randn(M, d, device="cuda")
    y = torch.randn(M, d, device="cuda")
    o = torch.empty(M, d, device="cuda")
    oa = torch.empty(M, d, device="cuda", dtype=torch.float16)
    g = torch.ones(d, device="cuda")
    b = torch.zeros(d, device="cuda")
    s = torch.cuda.Stream()
    gr = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(gr, stream=s):
        for _ in range(10):
            check(lib.fnmt_add_norm(ptr(x), ptr(y), ptr(g), ptr(b), 0, ptr(o), ptr(oa), _capi.F16, M,
                                    d, s.cuda_stream), "add_norm")
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 50
    print(f"rows {M}: {us:.1f} us  {M * d * 14 / us / 1e3:.0f} GB/s")
