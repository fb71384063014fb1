"""Multi-rank logic on CPU (gloo, world_size 2): corpus sharding covers every
sentence exactly once with balanced length mixes, the distributed translate
restores corpus order, and bench.py's timing reductions take the max over
ranks / sum of work."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2109_08003_b200.dispatch import restore, restore_flat, shard_indices


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shards_partition_the_corpus_with_equal_length_mix():
    rng = np.random.default_rng(0)
    lengths = np.clip(np.rint(rng.gamma(3, 8, size=10_001)), 1, 200).astype(int)
    for world in (1, 2, 4, 8):
        shards = [shard_indices(lengths, world, r) for r in range(world)]
        allidx = np.concatenate(shards)
        assert sorted(allidx.tolist()) == list(range(len(lengths)))
        tokens = [lengths[s].sum() for s in shards]
        assert max(tokens) - min(tokens) <= 200          # at most one sentence apart
    out = restore(shards, [[f"o{i}" for i in s] for s in shards], len(lengths))
    assert out == [f"o{i}" for i in range(len(lengths))]
    with pytest.raises(ValueError):
        restore(shards, [[1]] + [[0] * len(s) for s in shards[1:]], len(lengths))


def _worker(rank, world, port, rows, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2109_08003_b200.dispatch import translate_distributed

    # a stand-in engine: deterministic per-sentence function (reverse + rank-independent)
    def fake_engine(batch):
        return [list(reversed([int(x) for x in r])) for r in batch]

    got = translate_distributed(fake_engine, rows, dst=None)
    # bench.py reductions: max of per-rank time, sum of per-rank work
    import bench
    t_max, w_sum = bench.reduce_max_sum(dist, world, torch.device("cpu"), 1.0 + rank, 10.0 * (rank + 1))
    q.put((rank, got, t_max, w_sum))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_distributed_translate_and_reductions():
    rng = np.random.default_rng(1)
    rows = [rng.integers(4, 100, size=int(rng.integers(1, 30))).tolist() for _ in range(101)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, rows, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [list(reversed(r)) for r in rows]
    for rank, got, t_max, w_sum in results:
        assert got == want
        assert t_max == 2.0 and w_sum == 30.0


def test_restore_flat_matches_restore_and_native_order():
    """The flat gather's segment permutation equals the list restore, and the
    shards deal the native planner's permutation (fnmt_plan_batches) round-robin."""
    from paper_2109_08003_b200.engine import native_plan
    rng = np.random.default_rng(3)
    lengths = np.clip(np.rint(rng.gamma(3, 8, size=3001)), 1, 200).astype(int)
    perm, _ = native_plan(lengths, 3072, 64000)
    for world in (1, 2, 3, 8):
        shards = [shard_indices(lengths, world, r) for r in range(world)]
        for r in range(world):
            assert shards[r].tolist() == perm[r::world]
        outs = [[list(range(i % 7)) + [i] for i in s] for s in shards]
        ids = [np.concatenate([np.asarray(o, np.int32) for o in outs_r]) for outs_r in outs]
        lens = [np.array([len(o) for o in outs_r], np.int32) for outs_r in outs]
        flat, off = restore_flat(shards, ids, lens, len(lengths))
        want = restore(shards, outs, len(lengths))
        assert [flat[off[i]:off[i + 1]].tolist() for i in range(len(lengths))] == want
    with pytest.raises(ValueError):
        restore_flat(shards[:-1], ids[:-1], lens[:-1], len(lengths))


def _oracle_worker(rank, world, port, rows, q):
    """Real dispatch: each rank translates its shard with the CPU oracle of a
    tiny student (the computation every rank's engine performs), then the
    flat-buffer gather restores corpus order."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import nmt_oracle as O
    from paper_2109_08003_b200 import store as S
    from paper_2109_08003_b200.dispatch import translate_distributed
    cfg = S.ModelConfig(n_enc_layers=2, n_dec_layers=1, d_model=32, n_heads_enc=2,
                        n_heads_dec=1, ffn_dim_enc=64, ffn_dim_dec=32, vocab_size=120,
                        max_positions=64)
    a = O.arch_of(cfg)
    p = O.make_params(a, 5)

    def engine(batch):
        tok, valid = O.pad_rows([np.asarray(r, np.int64) for r in batch])
        return [list(map(int, o)) for o in O.greedy(a, p, tok, valid)]

    got0 = translate_distributed(engine, rows, dst=0)
    got_all = translate_distributed(engine, rows, dst=None)
    q.put((rank, got0, got_all, engine(rows) if rank == 0 else None))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_real_dispatch_oracle_engine():
    rng = np.random.default_rng(7)
    rows = [rng.integers(4, 120, size=int(rng.integers(1, 20))).tolist() for _ in range(37)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_oracle_worker, args=(r, 2, port, rows, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = sorted([q.get(timeout=300) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = results[0][3]
    assert results[0][1] == want and results[1][1] is None
    assert results[0][2] == want and results[1][2] == want
