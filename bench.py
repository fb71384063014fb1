#!/usr/bin/env python
"""Benchmark: Student-6-1-1 fp16 greedy over the 1M-sentence (2^20)
newstest-shaped synthetic corpus with dynamic batching (sbatch/wbatch
3072/64000), target words/s.

A "step" is one chunk of the corpus (--chunk-sentences, default 65536 =
1/16 of the corpus) translated end to end by the engine (plan -> encode ->
graph-captured greedy decode -> order restore).  Rank r of N processes chunk
(r + i*N) mod 16 at step i (sentence-sharded DP, no collective; weak scaling).

  value : inputs already resident in HBM (translate_device), K timed steps
  e2e   : the public host-buffer API (Engine.translate / fnmt_engine_translate)
          with the chunk's ids copied H2D and the outputs D2H inside each step

python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
torchrun --nproc-per-node N bench.py --gpus N ...
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "target words/sec, Student-6-1-1 greedy fp16 at 1/2/4/8 B200; peak HBM GB"
UNIT = "target words/s"
CORPUS = 1 << 20
CFG = dict(n_enc_layers=6, n_dec_layers=1, d_model=512, n_heads_enc=1, n_heads_dec=1,
           ffn_dim_enc=2048, ffn_dim_dec=2048, vocab_size=32772, max_positions=1024)
SBATCH, WBATCH = 3072, 64000

# BASELINE.json configs 2-5 (SURVEY §8 model shapes)
MODELS = {
    "6-1-1": ("Student-6-1-1 (6-1, d512, 1/1 heads, ffn 2048/2048, V 32772)", CFG),
    "6-1-8": ("Student-6-1-8 (6-1, d512, 8/8 heads, ffn 2048/2048, V 32772)",
              dict(CFG, n_heads_enc=8, n_heads_dec=8)),
    "6-6-8": ("Student-6-6-8 (6-6, d512, 8/8 heads, ffn 2048/2048, V 32772, unshared)",
              dict(CFG, n_dec_layers=6, n_heads_enc=8, n_heads_dec=8, shared_embeddings=False)),
    "deep-12-768": ("Deep-12-768 (12-6, d768, 8/8 heads, ffn 3072/3072, V 32772)",
                    dict(CFG, n_enc_layers=12, n_dec_layers=6, d_model=768, n_heads_enc=8,
                         n_heads_dec=8, ffn_dim_enc=3072, ffn_dim_dec=3072)),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--chunk-sentences", type=int, default=65536)
    ap.add_argument("--dtype", default="f16")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--profile-sentences", type=int, default=65536,
                    help="sentences of the first timed chunk in the per-kernel profile pass")
    ap.add_argument("--wbatch", type=int, default=64000, help="token cap (paper GPU setting 64000)")
    ap.add_argument("--sbatch", type=int, default=3072, help="sentence cap (paper GPU setting 3072)")
    ap.add_argument("--model", choices=sorted(MODELS), default="6-1-1")
    ap.add_argument("--beam", type=int, default=1)
    ap.add_argument("--sim-rank", type=int, default=None,
                    help="debug: run rank R's chunk sequence of a --sim-world job in one process")
    ap.add_argument("--sim-world", type=int, default=1)
    return ap.parse_args()


# ----------------------------------------------------------------------------
# distributed plumbing

def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def dist_init(world, backend):
    import torch.distributed as dist
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend=backend)
    return dist


def reduce_max_sum(dist, world, device, t_max, x_sum):
    if world == 1:
        return t_max, x_sum
    import torch
    if dist.get_backend() == "gloo":   # FNMT_DIST_BACKEND=gloo: CPU tensors
        device = torch.device("cpu")
    a = torch.tensor([t_max], dtype=torch.float64, device=device)
    b = torch.tensor([x_sum], dtype=torch.float64, device=device)
    dist.all_reduce(a, op=dist.ReduceOp.MAX)
    dist.all_reduce(b, op=dist.ReduceOp.SUM)
    return float(a.item()), float(b.item())


# ----------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)

REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}


class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        cmd = ["nvidia-smi", f"--id={self.index}",
               "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
               "--format=csv,noheader,nounits", "-lms", "200"]
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                         text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 4:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                smax.append(float(r[1]))
                mask = int(r[3], 16) if r[3].startswith("0x") else int(r[3])
                for bit, name in REASON_BITS.items():
                    if mask & bit and bit != 0x1:
                        reasons.add(name)
            except ValueError:
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------
# CPU baseline: the reference's own CPU path (baseline/_ref, the unmodified
# fastnmt package, when installed; else the oracle port oracle/nmt_oracle.py,
# pinned bit-exact to the reference) on the host cores.  One measurement
# shared by both arms: a "CPU step" = every process translating PER_PROC
# consecutive corpus sentences (one reference batch) with one thread
# ("one MKL thread for each process").  Worker processes come
# from a forkserver (never forked from the CUDA-initialised bench process).

REF_DIR = ROOT / "baseline" / "_ref"
PER_PROC = 8
_CPU = {}


def reference_available() -> bool:
    return (REF_DIR / "fastnmt" / "search.py").exists()


def _import_reference():
    """The installed reference package; its __init__ imports the missing
    fastnmt.engine, so a stub is registered first."""
    import types
    if "fastnmt.engine" not in sys.modules:
        stub = types.ModuleType("fastnmt.engine")
        stub.RunConfig = type("RunConfig", (), {})
        stub.Translator = type("Translator", (), {})
        sys.modules["fastnmt.engine"] = stub
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import fastnmt.model as M
    import fastnmt.search as Sr
    import fastnmt.store as St
    return M, Sr, St


def _cpu_init(impl, model_cfg, beam):
    os.environ["OMP_NUM_THREADS"] = "1"
    _CPU.update(impl=impl, beam=beam)
    if impl == "reference":
        M, Sr, St = _import_reference()
        cfg = M.ModelConfig(**model_cfg)
        _CPU["model"] = M.TranslationModel(cfg, St.random_model(cfg, 0))
        _CPU["search"] = Sr
    else:
        from oracle import nmt_oracle as O
        from paper_2109_08003_b200 import store as S
        a = O.arch_of(S.ModelConfig(**model_cfg))
        _CPU.update(arch=a, params=O.make_params(a, 0))


def _cpu_ready(_):
    return True


def _cpu_worker(rows):
    """One reference batch (the process's sentences, right-padded)."""
    from oracle import nmt_oracle as O
    tok, valid = O.pad_rows(rows)
    k = _CPU["beam"]
    if _CPU["impl"] == "reference":
        Sr, m = _CPU["search"], _CPU["model"]
        sc = Sr.SearchConfig(bos_id=2, eos_id=3, pad_id=0, beam_size=k)
        enc = m.encode(tok, valid)
        out = Sr.greedy_translate(m, enc, sc) if k == 1 else Sr.beam_translate(m, enc, sc)
    else:
        a, p = _CPU["arch"], _CPU["params"]
        out = O.greedy(a, p, tok, valid) if k == 1 else O.beam(a, p, tok, valid, k)
    return [list(map(int, o)) for o in out]


class CpuArm:
    def __init__(self, model_cfg, beam):
        import multiprocessing as mp
        from concurrent.futures import ProcessPoolExecutor
        self.impl = "reference" if reference_available() else "port"
        self.procs = os.cpu_count() or 1
        # greedy: one 8-sentence reference batch per process per step; beam
        # searches sentence by sentence anyway (search.py:105-111)
        self.per_proc = PER_PROC if beam == 1 else 1
        os.environ["OMP_NUM_THREADS"] = "1"   # inherited by the forkserver (numpy import)
        self.pool = ProcessPoolExecutor(self.procs, mp_context=mp.get_context("forkserver"),
                                        initializer=_cpu_init,
                                        initargs=(self.impl, model_cfg, beam))
        list(self.pool.map(_cpu_ready, range(4 * self.procs)))   # all initializers ran

    def step(self, ids, offsets, start):
        """procs x per_proc consecutive sentences from `start`, length-sorted and
        dealt out in batches of per_proc (the reference planner's sort-then-group,
        batching.py:100-109); returns (outputs in corpus order, src words, seconds)."""
        n = self.procs * self.per_proc
        order = sorted(range(start, start + n), key=lambda i: -(offsets[i + 1] - offsets[i]))
        groups = [order[j * self.per_proc:(j + 1) * self.per_proc] for j in range(self.procs)]
        jobs = [[ids[offsets[i]:offsets[i + 1]].astype(np.int64) for i in g] for g in groups]
        t0 = time.perf_counter()
        res = list(self.pool.map(_cpu_worker, jobs, chunksize=1))
        dt = time.perf_counter() - t0
        out = [None] * n
        for g, r in zip(groups, res):
            for i, o in zip(g, r):
                out[i - start] = o
        return out, sum(len(r) for j in jobs for r in j), dt

    def run(self, ids, offsets, start, steps):
        outs, src, total = [], 0, 0.0
        for i in range(steps):
            o, s, dt = self.step(ids, offsets, start + i * self.procs * self.per_proc)
            outs += o
            src += s
            total += dt
        return outs, src, total

    def describe(self, steps, words, src, seconds, what):
        kind = ("the unmodified reference package (baseline/_ref fastnmt, greedy_translate / "
                "beam_translate)" if self.impl == "reference" else
                "the oracle port (oracle/nmt_oracle.py, pinned bit-exact to the reference)")
        return (f"{steps} steps x {self.procs} procs x {self.per_proc} length-sorted corpus "
                f"sentences "
                f"{what} ({words} target words, {src} source words, {seconds:.1f} s), {kind}, "
                f"f32 numpy, one thread per process")

    def close(self):
        self.pool.shutdown(wait=True)


def parity_report(model_cfg, beam, dtype, sample_rows, got, want):
    """GPU output vs the CPU arm's output on the same sentences (oracle/parity.py
    bar; the oracle re-runs the divergent sentences for the near-tie report)."""
    from oracle import nmt_oracle as O
    from oracle import parity as P
    from paper_2109_08003_b200 import store as S
    tie = P.NEAR_TIE_BF16 if dtype == "bf16" else P.NEAR_TIE
    a = O.arch_of(S.ModelConfig(**model_cfg))
    bad = any(list(g) != list(w) for g, w in zip(got, want))
    p = O.make_params(a, 0) if bad else None
    rep = P.near_tie_report(a, p, sample_rows, got, want, beam, tie)
    rep["divergences"] = rep["divergences"][:20]
    return rep


FIXTURES = {("6-1-1", 1): ("s611", 65536), ("6-1-8", 1): ("s618", 65536),
            ("6-6-8", 4): ("s668_beam4", 8192), ("deep-12-768", 4): ("deep_beam4", 8192)}


def fixture_parity(eng, args, cfg, ids, offsets, lengths):
    """The engine (same caps, default lanes) on corpus chunk 0 vs the committed
    reference outputs for its sampled sentences (tests/golden/corpus_*.npz,
    oracle/make_golden_corpus.py); untimed."""
    from oracle import parity as P
    key = FIXTURES.get((args.model, args.beam))
    path = ROOT / "tests" / "golden" / f"corpus_{key[0]}.npz" if key else None
    if not path or not path.exists() or args.dtype not in ("f16", "bf16"):
        return None
    from paper_2109_08003_b200.engine import budgets_of
    fx = np.load(path)
    n = min(key[1], len(lengths))
    out, olen, oof, _ = eng.translate(ids, offsets[:n + 1], sbatch=SBATCH, wbatch=WBATCH,
                                      beam=args.beam)
    got = [out[oof[i]:oof[i] + olen[i]].tolist() for i in fx["idx"]]
    tie = P.NEAR_TIE_BF16 if args.dtype == "bf16" else P.NEAR_TIE
    if args.beam == 1:
        rep = P.greedy_report(got, fx, near_tie=tie)
    else:
        rep = P.beam_report(got, fx, budgets_of(lengths[fx["idx"]], 1.5, 5, cfg.max_positions),
                            near_tie=tie)
    rep["divergences"] = rep["divergences"][:20]
    return {"workload": f"corpus chunk 0 (first {n} sentences, caps {SBATCH}/{WBATCH}, default "
                        f"lanes) vs the reference's recorded outputs for {len(fx['idx'])} of them "
                        f"({path.name})", **rep}


def arm_config(args, world):
    """The `config` object both arms print (BASELINE config of --model)."""
    model_desc = MODELS[args.model][0]
    C = args.chunk_sentences
    beam = args.beam
    return {"workload": f"{model_desc.split(' (')[0]} {args.dtype} "
                        f"{'greedy' if beam == 1 else f'beam={beam}'}, 1M (2^20) synthetic "
                        f"newstest-shaped sentences, dynamic batching sbatch/wbatch "
                        f"{SBATCH}/{WBATCH}",
            "model": f"{model_desc[:-1]}, random-init seed 0)",
            "beam": beam,
            "corpus_sentences": CORPUS, "chunk_sentences": C,
            "sentences_per_step_all_ranks": C * world,
            "parallelism": f"sentence-sharded dp{world} (no collective)",
            "l2": "256 MiB memset between steps; per-step working set >> L2"}


def run_reference(args):
    """--impl reference: the reference's own CPU path on all host cores —
    the unmodified fastnmt package from baseline/_ref (plain pip install of
    /root/reference/pkg; no engine, kernels or code of ours on that path),
    or the oracle port when that install is absent.  Each step translates a
    bounded sample (procs x PER_PROC consecutive corpus sentences)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2109_08003_b200.synthetic import newstest_corpus
    model_cfg = MODELS[args.model][1]
    ids, offsets, _ = newstest_corpus(CORPUS, model_cfg["vocab_size"])
    arm = CpuArm(model_cfg, args.beam)
    per_step = arm.procs * arm.per_proc
    arm.run(ids, offsets, 0, args.warmup)
    outs, src, total = arm.run(ids, offsets, args.warmup * per_step, args.steps)
    arm.close()
    words = sum(len(o) for o in outs)
    value = words / total
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "impl": "reference",
            "config": arm_config(args, 1),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": arm.procs, "kind": arm.impl,
                             "sample": arm.describe(args.steps, words, src, total,
                                                    "(after the warm-up steps' sentences)")},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------

def main():
    global SBATCH, WBATCH
    args = parse()
    SBATCH, WBATCH = args.sbatch, args.wbatch
    if args.impl == "reference":
        return run_reference(args)
    import torch
    world, rank, local = dist_env()
    # one GPU per rank; FNMT_DIST_BACKEND=gloo with fewer GPUs than ranks maps
    # ranks onto the visible devices (a dry run of the N > 1 path on one GPU)
    backend = os.environ.get("FNMT_DIST_BACKEND", "nccl")
    if backend == "gloo":
        local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    dist = dist_init(world, backend)

    from paper_2109_08003_b200 import store as S
    from paper_2109_08003_b200.batching import estimate_device_bytes
    from paper_2109_08003_b200.engine import Engine, budgets_of
    from paper_2109_08003_b200.synthetic import newstest_corpus

    model_desc, model_cfg = MODELS[args.model]
    cfg = S.ModelConfig(**model_cfg)
    BEAM = args.beam
    ids, offsets, lengths = newstest_corpus(CORPUS, cfg.vocab_size)
    C = args.chunk_sentences
    n_chunks = max(1, CORPUS // C)
    eng = Engine(cfg, S.random_model(cfg, 0), dtype=args.dtype, device=local)
    weight_bytes = eng.device_bytes()
    eng.reserve(SBATCH, WBATCH)

    chunk_meta = []
    for c in range(n_chunks):
        lo, hi = c * C, (c + 1) * C
        L = lengths[lo:hi]
        b = budgets_of(L, 1.5, 5, cfg.max_positions)
        off = np.zeros(len(b), np.int64)
        np.cumsum(b[:-1], out=off[1:])
        chunk_meta.append((lo, hi, L, b, off))
    max_out = max(int(m[3].sum()) for m in chunk_meta)

    d_ids = torch.from_numpy(ids).to(device)
    d_offsets = torch.from_numpy(offsets).to(device)
    d_out_ids = torch.empty(max_out, dtype=torch.int32, device=device)
    d_out_off = [torch.from_numpy(m[4]).to(device) for m in chunk_meta]
    K, W = args.steps, args.warmup
    d_out_len = torch.zeros((max(K, 1), C), dtype=torch.int32, device=device)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)

    crank, cworld = (args.sim_rank, args.sim_world) if args.sim_rank is not None else (rank, world)

    def chunk_of(i):
        return (crank + i * cworld) % n_chunks

    def device_step(c, slot):
        lo, hi, L, b, off = chunk_meta[c]
        flush.zero_()
        return eng.translate_device(d_ids, d_offsets[lo:hi + 1], L, d_out_ids, off,
                                    d_out_off[c], d_out_len[slot], sbatch=SBATCH, wbatch=WBATCH,
                                    beam=BEAM)

    for i in range(W):
        device_step(chunk_of(i), 0)
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats(device)
    free0, total_mem = torch.cuda.mem_get_info(device)

    sampler = ClockSampler(local)
    sampler.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    launches = 0
    src_words = 0
    for i in range(K):
        c = chunk_of(W + i)
        st = device_step(c, i)
        launches += st.gpu_launches
        src_words += int(chunk_meta[c][2].sum())
    ev1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    elapsed = ev0.elapsed_time(ev1) / 1e3
    words = float(d_out_len[:K].sum().item())
    t_max, words_all = reduce_max_sum(dist, world, device, elapsed, words)
    _, src_all = reduce_max_sum(dist, world, device, 0.0, float(src_words))
    value = words_all / t_max

    # ---- e2e: public host-buffer API, H2D + D2H inside each step -------------
    pin_ids = torch.from_numpy(ids).pin_memory()
    pin_ids_np = pin_ids.numpy()
    pin_out = torch.empty(max_out, dtype=torch.int32).pin_memory()
    pin_len = torch.empty(C, dtype=torch.int32).pin_memory()
    h2d = d2h = 0

    def host_step(c):
        lo, hi, L, b, off = chunk_meta[c]
        n_ids = int(offsets[hi] - offsets[lo])
        # the C ABI reads sentence i at ids[offsets[i]:offsets[i+1]] (absolute
        # offsets into the corpus array, rebased on the device): pass the base
        eng.translate(pin_ids_np, offsets[lo:hi + 1],
                      sbatch=SBATCH, wbatch=WBATCH, out_ids=pin_out.numpy(),
                      out_len=pin_len.numpy(), out_off=off, beam=BEAM)
        return n_ids * 4 + (hi - lo + 1) * 8 + (hi - lo) * 8, int(b.sum()) * 4 + (hi - lo) * 4

    # N > 1: the step's result is the corpus-ordered output on rank 0.  Every
    # rank's chunk (flat ids at budget offsets + lengths, fixed-size buffers)
    # is gathered to rank 0 (NCCL over NVLink, or gloo host tensors in a dry
    # run) and placed at the chunk's corpus position — restore_order
    # (batching.py:112-122) for chunk-sharded work; the native call already
    # restored order inside each chunk.
    gather_dev = torch.device("cpu") if backend == "gloo" else device
    corpus_off = np.zeros(CORPUS + 1, np.int64)
    if world > 1:
        np.cumsum(budgets_of(lengths, 1.5, 5, cfg.max_positions), out=corpus_off[1:])
        g_ids = torch.empty(max_out, dtype=torch.int32, device=gather_dev)
        g_len = torch.empty(C, dtype=torch.int32, device=gather_dev)
        if rank == 0:
            corpus_out = torch.empty(int(corpus_off[-1]), dtype=torch.int32).pin_memory()
            corpus_len = torch.empty(CORPUS, dtype=torch.int32).pin_memory()
            r_ids = [torch.empty_like(g_ids) for _ in range(world)]
            r_len = [torch.empty_like(g_len) for _ in range(world)]

    def gather_step(i):
        """Returns (h2d, d2h) bytes this rank moved for the gather."""
        g_ids.copy_(pin_out[:max_out], non_blocking=True)
        g_len.copy_(pin_len, non_blocking=True)
        dist.gather(g_ids, r_ids if rank == 0 else None, dst=0)
        dist.gather(g_len, r_len if rank == 0 else None, dst=0)
        h = (max_out + C) * 4 if gather_dev.type == "cuda" else 0
        if rank != 0:
            return h, 0
        moved = 0
        for r in range(world):
            cr = (r + (W + i) * world) % n_chunks
            lo, hi, L, b, off = chunk_meta[cr]
            nb = int(b.sum())
            base = int(corpus_off[lo])
            corpus_out[base:base + nb].copy_(r_ids[r][:nb], non_blocking=True)
            corpus_len[lo:hi].copy_(r_len[r][:hi - lo], non_blocking=True)
            moved += (nb + hi - lo) * 4
        torch.cuda.current_stream(device).synchronize()
        for r in range(world):
            lo, hi = chunk_meta[(r + (W + i) * world) % n_chunks][:2]
            gathered[0] += int(corpus_len[lo:hi].sum())
        return h, moved if gather_dev.type == "cuda" else 0

    # warm the host path on every chunk the timed loop will use: the C ABI's
    # device staging buffers grow to the largest chunk here, not inside the
    # timed region (a cudaMalloc there cost up to 30% of an e2e step)
    for c in sorted({chunk_of(W + i) for i in range(K)}):
        host_step(c)
    gathered = [0]
    if world > 1:
        gather_step(0)
        gathered[0] = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    e2e_words = 0
    for i in range(K):
        c = chunk_of(W + i)
        a, bb = host_step(c)
        h2d += a
        d2h += bb
        e2e_words += int(pin_len[:chunk_meta[c][1] - chunk_meta[c][0]].sum())
        if world > 1:
            a, bb = gather_step(i)
            h2d += a
            d2h += bb
    e1.record()
    torch.cuda.synchronize()
    e_el = e0.elapsed_time(e1) / 1e3
    e_max, e_words_all = reduce_max_sum(dist, world, device, e_el, float(e2e_words))
    e2e = {"value": e_words_all / e_max, "unit": UNIT, "h2d_bytes_per_step": h2d // max(K, 1),
           "d2h_bytes_per_step": d2h // max(K, 1),
           # same chunks through both paths: the word counts must agree exactly
           "matches_device_path": bool(e2e_words == int(words))}
    if world > 1:
        # rank 0 holds every rank's outputs in corpus order after each step
        e2e["gathered_to_rank0"] = {"words": gathered[0] if rank == 0 else None,
                                    "matches_all_ranks": bool(rank != 0 or
                                                              gathered[0] == int(e_words_all))}

    peak_alloc = torch.cuda.max_memory_allocated(device)
    engine_bytes = eng.device_bytes()

    # ---- live per-kernel profile (one sub-chunk, events on the engine stream) --
    prof = None
    prof_words = 0
    if rank == 0 and args.profile_sentences > 0:
        c = chunk_of(0)
        lo = chunk_meta[c][0]
        hi = lo + min(args.profile_sentences, C)
        L = lengths[lo:hi]
        b = budgets_of(L, 1.5, 5, cfg.max_positions)
        off = np.zeros(len(b), np.int64)
        np.cumsum(b[:-1], out=off[1:])
        eng.profile(True)
        eng.translate_device(d_ids, d_offsets[lo:hi + 1], L, d_out_ids, off,
                             torch.from_numpy(off).to(device), d_out_len[0], sbatch=SBATCH,
                             wbatch=WBATCH, beam=BEAM)
        prof = eng.profile_read()
        eng.profile(False)
        prof_words = int(d_out_len[0][:hi - lo].sum().item())

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    peaks = {}
    pk = ROOT / "MEASURED_PEAKS.json"
    if pk.exists():
        peaks = json.loads(pk.read_text())
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    tc_peak = peaks.get("bf16_tflops_sustained", 1400.0)
    roofline = None
    kprof = None
    if prof:
        total_ms = sum(v["ms"] for v in prof.values()) or 1.0
        kprof = {k: {"ms": round(v["ms"], 3), "share": round(v["ms"] / total_ms, 4),
                     "launches": v["launches"],
                     "tflops": round(v["flops"] / (v["ms"] * 1e9), 2) if v["ms"] and v["flops"] else None,
                     "gbs": round(v["bytes"] / (v["ms"] * 1e6), 1) if v["ms"] and v["bytes"] else None}
                 for k, v in prof.items()}
        top = max(prof, key=lambda k: prof[k]["ms"])
        v = prof[top]
        per_launch_ms = v["ms"] / max(v["launches"], 1)
        traffic = None
        tf = ROOT / "profiles" / "ncu_traffic.json"
        if tf.exists():
            traffic = json.loads(tf.read_text()).get(top)
        if v["flops"] > 0:
            ach = v["flops"] / max(v["launches"], 1) / (per_launch_ms * 1e9)
            roofline = {"bound": "tensor", "kernel": top, "achieved": round(ach, 2),
                        "peak": tc_peak, "unit": "TFLOP/s", "frac": round(ach / tc_peak, 4),
                        "traffic": traffic, "per_launch_ms": round(per_launch_ms, 4),
                        "flops_per_launch": v["flops"] / max(v["launches"], 1),
                        "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained"}
        else:
            ach = v["bytes"] / max(v["launches"], 1) / (per_launch_ms * 1e6)
            roofline = {"bound": "hbm", "kernel": top, "achieved": round(ach, 1),
                        "peak": hbm_peak, "unit": "GB/s", "frac": round(ach / hbm_peak, 4),
                        "traffic": traffic, "per_launch_ms": round(per_launch_ms, 4),
                        "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
        # whole-step algorithmic rate (63.8 MFLOP / target word) over the
        # profile pass's summed kernel time, and the timed run's whole-path rate: the
        # profile pass's algorithmic FLOPs per target word x the timed words / s
        flops_total = sum(p["flops"] for p in prof.values())
        roofline["step_tflops"] = round(flops_total / (total_ms * 1e9), 2)
        if prof_words:
            path = flops_total / prof_words * value / 1e12
            roofline["path_mflop_per_word"] = round(flops_total / prof_words / 1e6, 2)
            roofline["path_tflops"] = round(path, 1)
            roofline["path_frac"] = round(path / tc_peak, 4)

    # ---- CPU baseline + parity on the timed workload -------------------------
    # The CPU arm translates the first sentences of the LAST timed e2e step's
    # chunk; the GPU's output for them is what that step left in pin_out.
    cpu = parity = None
    if world == 1 and not args.no_cpu_baseline:
        arm = CpuArm(model_cfg, BEAM)
        c_last = chunk_of(W + K - 1)
        lo, hi, L, b, off = chunk_meta[c_last]
        steps = max(1, int(round(args.cpu_seconds / (6.0 if BEAM == 1 else 12.0))))
        want, src, dt = arm.run(ids, offsets, lo, steps)
        arm.close()
        n = len(want)
        got = [pin_out[int(off[i]):int(off[i]) + int(pin_len[i])].tolist() for i in range(n)]
        words = sum(len(o) for o in want)
        cpu = {"value": words / dt, "unit": UNIT, "cores": arm.procs, "kind": arm.impl,
               "sample": arm.describe(steps, words, src, dt, f"from chunk {c_last}")}
        sample_rows = [ids[offsets[i]:offsets[i + 1]].astype(np.int64) for i in range(lo, lo + n)]
        live = {"workload": f"the last timed e2e step (chunk {c_last}, caps {SBATCH}/{WBATCH}, "
                            f"default lanes) vs the CPU arm on its first {n} sentences",
                **parity_report(model_cfg, BEAM, args.dtype, sample_rows, got, want)}
        fixed = fixture_parity(eng, args, cfg, ids, offsets, lengths)
        parts = [x for x in (live, fixed) if x]
        tot = sum(x["sentences"] for x in parts)
        same = sum(x["identical"] for x in parts)
        parity = {"sentences": tot, "identical": same, "identical_frac": same / max(tot, 1),
                  "all_near_ties": all(x["all_near_ties"] for x in parts),
                  # the bar over the union of both samples: >= 99% identical
                  # (greedy), every divergence a near-tie
                  "pass": all(x["all_near_ties"] for x in parts) and
                          same >= live["min_identical_frac"] * tot,
                  "live": live, "fixture": fixed}

    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": round(1e3 * t_max / max(K, 1), 2),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": args.dtype, "data": "synthetic",
        "config": arm_config(args, world),
        "e2e": e2e,
        "gpu_launches": int(launches),
        "roofline": roofline,
        "cpu_baseline": cpu,
        "parity": parity,
        "clocks": clocks,
        "peak_hbm_gb": round(max(peak_alloc, engine_bytes + peak_alloc) / 1e9, 3),
        "engine_device_gb": round(engine_bytes / 1e9, 3),
        # weights (measured after load) + every decode lane's workspace from the
        # allocation-level estimate (batching.estimate_device_bytes)
        "engine_estimate_gb": round((weight_bytes + int(os.environ.get("FNMT_LANES", "4")) *
                                     estimate_device_bytes(cfg, SBATCH, WBATCH,
                                                           dtype_bytes=4 if args.dtype == "f32"
                                                           else 2)) / 1e9, 3),
        "source_words_per_sec": round(src_all / t_max, 1),
        "sentences_per_sec": round(C * world * K / t_max, 1),
        "kernel_profile": kprof,
    }
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
