"""Length-sorted dynamic batching (host-side scheduler).

API-compatible with the reference's batching module (batching.py:35-165):
``DecodeLimits``, ``Batch``, ``BatchPlan``, ``sort_by_length_desc``,
``form_batches``, ``plan_batches``, ``restore_order``,
``estimate_peak_memory`` and ``IntegrityError``.  The CUDA engine runs the
same planner natively (csrc/engine.cu ``plan_batches``) for corpus
translation; this module serves callers that drive batches themselves.

GPU caps from the paper: sbatch/wbatch 3072/64000.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

GPU_SBATCH, GPU_WBATCH = 3072, 64000


class IntegrityError(ValueError):
    """Outputs do not line up with the batch plan."""


@dataclass(frozen=True)
class DecodeLimits:
    sbatch: int = 128
    wbatch: int = 2048

    def __post_init__(self):
        if self.sbatch < 1 or self.wbatch < 1:
            raise ValueError("sbatch and wbatch must be >= 1")


@dataclass(frozen=True)
class Batch:
    indices: tuple
    max_len: int
    oversize: bool = False

    @property
    def padded_shape(self):
        return (len(self.indices), self.max_len)


@dataclass(frozen=True)
class BatchPlan:
    batches: tuple
    permutation: tuple

    @property
    def n_items(self) -> int:
        return len(self.permutation)


def sort_by_length_desc(lengths) -> list:
    return sorted(range(len(lengths)), key=lambda i: -lengths[i])


def form_batches(sorted_lengths, limits: DecodeLimits) -> list:
    lengths = list(sorted_lengths)
    for a, b in zip(lengths, lengths[1:]):
        if a < b:
            raise ValueError("lengths must be sorted in descending order")
    out, members, longest = [], [], 0
    for pos, n in enumerate(lengths):
        grow = len(members) + 1
        if members and grow <= limits.sbatch and grow * longest <= limits.wbatch:
            members.append(pos)
            continue
        if members:
            out.append(Batch(tuple(members), longest, oversize=longest > limits.wbatch))
        members, longest = [pos], n
    if members:
        out.append(Batch(tuple(members), longest, oversize=longest > limits.wbatch))
    return out


def plan_batches(lengths, limits: DecodeLimits) -> BatchPlan:
    order = sort_by_length_desc(lengths)
    groups = form_batches([lengths[i] for i in order], limits)
    batches = tuple(Batch(tuple(order[p] for p in g.indices), g.max_len, g.oversize)
                    for g in groups)
    return BatchPlan(batches=batches, permutation=tuple(i for b in batches for i in b.indices))


def restore_order(outputs, plan: BatchPlan) -> list:
    outputs = list(outputs)
    if len(outputs) != plan.n_items:
        raise IntegrityError(f"got {len(outputs)} outputs for a plan of {plan.n_items} sentences")
    restored = [None] * plan.n_items
    for value, original in zip(outputs, plan.permutation):
        restored[original] = value
    return restored


BASE_OVERHEAD_BYTES = 8 << 20
SLACK_FACTOR = 1.5


def estimate_peak_memory(plan: BatchPlan, cfg, max_out_len: int) -> int:
    """The reference's f32 CPU upper bound (batching.py:134-165), kept for
    API parity; see :func:`estimate_device_bytes` for the GPU engine."""
    if not plan.batches:
        return BASE_OVERHEAD_BYTES
    sizes = [(len(b.indices), b.max_len) for b in plan.batches]
    n_max = max(n for n, _ in sizes)
    nl = max(n * L for n, L in sizes)
    nll = max(n * L * L for n, L in sizes)
    ncache = max(n * (L + max_out_len) for n, L in sizes)
    d = cfg.d_model
    heads = max(cfg.n_heads_enc, cfg.n_heads_dec)
    ffn = max(cfg.ffn_dim_enc, cfg.ffn_dim_dec, d)
    live = (nl * d * (cfg.n_enc_layers + 5) + nll * heads * 3 + nl * ffn * 2
            + ncache * d * cfg.n_dec_layers * 2 + n_max * cfg.vocab_size * 2) * 4
    return BASE_OVERHEAD_BYTES + math.ceil(SLACK_FACTOR * live)


def estimate_device_bytes(cfg, sbatch: int, wbatch: int, dtype_bytes: int = 2,
                          ratio: float = 1.5, offset: int = 5) -> int:
    """One decode lane's workspace at the given caps, allocation by allocation
    as csrc/engine.cu Engine::reserve_for / Engine::reserve make it (greedy;
    the folded single-head layout when the engine uses it).  The engine's total
    is the weights plus this per lane (tests/test_gpu_memory.py checks it)."""
    d, fe, fd = cfg.d_model, cfg.ffn_dim_enc, max(cfg.ffn_dim_dec, 8)
    es = dtype_bytes
    tok = max(wbatch, cfg.max_positions)
    rows = max(sbatch, 1)
    pool = max(math.ceil(ratio * wbatch) + (offset + 1) * sbatch, cfg.max_positions)
    folded = es != 4 and cfg.n_heads_dec == 1 and d % 256 == 0
    act = lambda n: 0 if es == 4 else es * n   # noqa: E731  (fp32 engines alias the f32 buffer)
    enc = 4 * tok * 2 + 4 * (rows + 1) + 4 * rows * 3 + 4 * tok * d * 2 + act(tok * d)
    enc += es * tok * 3 * d + es * tok * d + es * tok * fe
    row_w = 2 * d + 8 if folded else 2 * d
    dec = cfg.n_dec_layers * (es * tok * row_w + es * pool * row_w)
    step = 4 * rows * d * 2 + act(rows * d) + es * rows * (3 * d + d + d + fd)
    step += 8 * rows + 4 * rows * 3 + rows + 4 * pool + 16
    return enc + dec + step