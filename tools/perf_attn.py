"""Encoder attention microbenchmark (fnmt_attention, the engine's varlen
tensor-core kernel): Student-6-1-1 shape (1 head, d 512) over a batch of
equal-length sequences read from the packed q|k|v layout, timed with CUDA
events over graph-captured launches.  Prints us per launch and the achieved
q, k, v, out bytes / time.

Usage: python tools/perf_attn.py [seq_len] [n_seq] [heads]"""

import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2109_08003_b200 import _capi  # noqa: E402
from paper_2109_08003_b200._capi import check, lib, ptr  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 24
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64000 // L
H = int(sys.argv[3]) if len(sys.argv) > 3 else 1
d = 512
dev = torch.device("cuda")
qkv = torch.randn(B * L, 3 * d, device=dev).half()
out = torch.empty(B * L, d, device=dev).half()
start = torch.arange(0, B * L, L, dtype=torch.int32, device=dev)
lens = torch.full((B,), L, dtype=torch.int32, device=dev)
s = torch.cuda.Stream()
q, k, v = qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:]
g = torch.cuda.CUDAGraph()
torch.cuda.synchronize()
with torch.cuda.graph(g, stream=s):
    for _ in range(10):
        check(lib.fnmt_attention(ptr(q), 3 * d, ptr(k), ptr(v), 3 * d, ptr(out), d, _capi.F16, H,
                                 d // H, ptr(start), ptr(lens), ptr(start), ptr(lens), L, B, L, L,
                                 s.cuda_stream), "attention")
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    g.replay()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / 50
print(f"L={L} B={B} heads={H}: {us:.1f} us  {B * L * d * 2 * 4 / us / 1e6:.0f} GB/s")
