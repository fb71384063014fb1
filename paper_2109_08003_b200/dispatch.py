"""Multi-GPU corpus dispatch: sentences are independent, so
the corpus is sharded across ranks with no data-path collective.

* ``shard_indices`` — length-sort the corpus once (the stable descending
  order of batching.py:68-70) and deal sentences round-robin, so every rank
  gets the same length mix (equal work per GPU, no straggler rank).
* ``translate_distributed`` — inside an initialised ``torch.distributed``
  group (one process per GPU, NCCL or gloo), every rank translates its shard
  with its own engine, then the per-rank outputs are gathered with a single
  object gather to ``dst`` and put back in corpus order (batching.py:112-122).
  The gather is host-side result collection, not part of the hot path.
"""

from __future__ import annotations

from typing import Callable, Optional, Sequence

import numpy as np


def shard_indices(lengths: Sequence[int], world: int, rank: int) -> np.ndarray:
    """Sentence indices owned by ``rank``: position i of the length-sorted
    order goes to rank i mod world."""
    lengths = np.asarray(lengths)
    order = np.argsort(-lengths, kind="stable")
    return order[rank::world]


def restore(shards: Sequence[np.ndarray], outputs: Sequence[Sequence], n: int) -> list:
    """Inverse of the sharding: outputs[r][j] belongs to sentence shards[r][j]."""
    res: list = [None] * n
    for idx, outs in zip(shards, outputs):
        if len(idx) != len(outs):
            raise ValueError("shard output count does not match its index list")
        for i, o in zip(idx, outs):
            res[int(i)] = o
    if any(r is None for r in res):
        raise ValueError("some sentences were not translated")
    return res


def translate_distributed(translate_fn: Callable[[list], list], rows: Sequence, group=None,
                          dst: Optional[int] = 0) -> Optional[list]:
    """Translate ``rows`` (list of id sequences, identical on every rank)
    across the ranks of ``group``.  ``translate_fn(list_of_rows) -> list`` is
    this rank's engine call (e.g. ``Engine`` / ``translate_ids``).  Returns the
    outputs in corpus order on ``dst`` (or on every rank if dst is None)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lengths = [len(r) for r in rows]
    mine = shard_indices(lengths, world, rank)
    outs = translate_fn([rows[int(i)] for i in mine])
    gathered = [None] * world
    if dst is None:
        dist.all_gather_object(gathered, outs, group=group)
    else:
        dist.gather_object(outs, gathered if rank == dst else None, dst=dst, group=group)
        if rank != dst:
            return None
    shards = [shard_indices(lengths, world, r) for r in range(world)]
    return restore(shards, gathered, len(rows))
