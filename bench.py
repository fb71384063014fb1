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
    ap.add_argument("--profile-sentences", type=int, default=16384)
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
# CPU baseline: the oracle port (oracle/nmt_oracle.py) on the host cores

_CPU_STATE = {}


def _cpu_worker(rows):
    from oracle import nmt_oracle as O
    a, p, k = _CPU_STATE["arch"], _CPU_STATE["params"], _CPU_STATE["beam"]
    tok, valid = O.pad_rows(rows)
    out = O.greedy(a, p, tok, valid) if k == 1 else O.beam(a, p, tok, valid, k)
    return sum(len(o) for o in out), sum(len(r) for r in rows)


def cpu_run(rows_per_proc, procs):
    """Translate procs x rows_per_proc sentences, one process per core (fork),
    OMP_NUM_THREADS=1 (PAPER.md:179 'one MKL thread for each process')."""
    import multiprocessing as mp
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(procs) as pool:
        res = pool.map(_cpu_worker, rows_per_proc)
    dt = time.perf_counter() - t0
    return sum(r[0] for r in res), sum(r[1] for r in res), dt


def cpu_setup(model_cfg=None, beam=1):
    """The selected model (BASELINE config of --model) with random_model(cfg, 0)
    weights, greedy or beam as --beam says."""
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import nmt_oracle as O
    from paper_2109_08003_b200 import store as S
    a = O.arch_of(S.ModelConfig(**(model_cfg or CFG)))
    _CPU_STATE["arch"] = a
    _CPU_STATE["params"] = O.make_params(a, 0)
    _CPU_STATE["beam"] = beam


def cpu_sample(ids, offsets, start, procs, per_proc):
    rows, k = [], start
    for _ in range(procs):
        grp = []
        for _ in range(per_proc):
            grp.append(ids[offsets[k]:offsets[k + 1]].astype(np.int64))
            k += 1
        rows.append(grp)
    return rows, k


def cpu_baseline(ids, offsets, seconds, model_cfg=None, beam=1):
    cpu_setup(model_cfg, beam)
    procs = os.cpu_count() or 1
    # calibrate per-process sample size to ~`seconds` of work (~55 words/s/core for
    # Student-6-1-1 greedy; the beam / larger configs run ~15-20x slower)
    rate = 55.0 if (beam == 1 and (model_cfg or CFG)["n_dec_layers"] == 1) else 3.0
    per_proc = max(1, int(seconds * rate / 41.25 / 1.5))
    rows, _ = cpu_sample(ids, offsets, 0, procs, per_proc)
    words, src, dt = cpu_run(rows, procs)
    return {"value": words / dt, "unit": UNIT, "cores": procs, "kind": "port",
            "sample": f"{procs} procs x {per_proc} sentences of the synthetic corpus "
                      f"({words} target words, {src} source words, {dt:.1f} s), oracle/nmt_oracle.py "
                      f"f32 numpy {'greedy' if beam == 1 else f'beam {beam}'}, one thread per process"}


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
    """--impl reference: the reference algorithm's CPU path (oracle port of
    fastnmt, /root/reference is not on the GPU box) on all host cores."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2109_08003_b200.synthetic import newstest_corpus
    model_cfg = MODELS[args.model][1]
    ids, offsets, _ = newstest_corpus(CORPUS, model_cfg["vocab_size"])
    cpu_setup(model_cfg, args.beam)
    procs = os.cpu_count() or 1
    per_proc = 2 if args.beam == 1 and model_cfg["n_dec_layers"] == 1 else 1
    k = 0
    for _ in range(args.warmup):
        rows, k = cpu_sample(ids, offsets, k, procs, 1)
        cpu_run(rows, procs)
    words = src = 0
    total = 0.0
    for _ in range(args.steps):
        rows, k = cpu_sample(ids, offsets, k, procs, per_proc)
        w, s, dt = cpu_run(rows, procs)
        words += w
        src += s
        total += dt
    value = words / total
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "impl": "reference",
            "config": arm_config(args, 1),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "port",
                             "sample": f"{args.steps} steps x {procs} procs x {per_proc} sentences "
                                       f"of the same corpus ({words} target words), the "
                                       f"reference algorithm (oracle/nmt_oracle.py, f32 numpy, "
                                       f"pinned to the reference) on the host cores"},
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
    from paper_2109_08003_b200.engine import Engine, budgets_of
    from paper_2109_08003_b200.synthetic import newstest_corpus

    model_desc, model_cfg = MODELS[args.model]
    cfg = S.ModelConfig(**model_cfg)
    BEAM = args.beam
    ids, offsets, lengths = newstest_corpus(CORPUS, cfg.vocab_size)
    C = args.chunk_sentences
    n_chunks = max(1, CORPUS // C)
    eng = Engine(cfg, S.random_model(cfg, 0), dtype=args.dtype, device=local)
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

    # warm the host path on every chunk the timed loop will use: the C ABI's
    # device staging buffers grow to the largest chunk here, not inside the
    # timed region (a cudaMalloc there cost up to 30% of an e2e step)
    for c in sorted({chunk_of(W + i) for i in range(K)}):
        host_step(c)
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
    e1.record()
    torch.cuda.synchronize()
    e_el = e0.elapsed_time(e1) / 1e3
    e_max, e_words_all = reduce_max_sum(dist, world, device, e_el, float(e2e_words))
    e2e = {"value": e_words_all / e_max, "unit": UNIT, "h2d_bytes_per_step": h2d // max(K, 1),
           "d2h_bytes_per_step": d2h // max(K, 1),
           # same chunks through both paths: the word counts must agree exactly
           "matches_device_path": bool(e2e_words == int(words))}

    peak_alloc = torch.cuda.max_memory_allocated(device)
    engine_bytes = eng.device_bytes()

    # ---- live per-kernel profile (one sub-chunk, events on the engine stream) --
    prof = None
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
        # whole-step algorithmic rate (63.8 MFLOP / target word)
        roofline["step_tflops"] = round(sum(p["flops"] for p in prof.values()) / (total_ms * 1e9), 2)

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(ids, offsets, args.cpu_seconds, model_cfg, BEAM)

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
        "clocks": clocks,
        "peak_hbm_gb": round(max(peak_alloc, engine_bytes + peak_alloc) / 1e9, 3),
        "engine_device_gb": round(engine_bytes / 1e9, 3),
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
