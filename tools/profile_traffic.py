"""The bench's profile pass, alone, for ncu: Student-6-1-1 fp16 greedy over
corpus chunk 0 (the first 65 536 sentences of the 2^20 corpus, caps
3072/64000), engine profiler on (one lane, un-captured launches), bracketed
by cudaProfilerStart/Stop so `ncu --profile-from-start off` sees exactly
these launches.  Writes the engine's per-launch log (class, event ms,
algorithmic FLOPs / bytes, launch order) to gpurun_out/prof_log_<tag>.npz;
tools/traffic_ratio.py matches it against the ncu CSV launch by launch.

Usage: python tools/profile_traffic.py [tag] [n_sentences] [model] [beam] [dtype]"""

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2109_08003_b200 import store as S  # noqa: E402
from paper_2109_08003_b200.engine import Engine, budgets_of  # noqa: E402
from paper_2109_08003_b200.synthetic import newstest_corpus  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
model = sys.argv[3] if len(sys.argv) > 3 else "6-1-1"
beam = int(sys.argv[4]) if len(sys.argv) > 4 else 1
dtype = sys.argv[5] if len(sys.argv) > 5 else "f16"
_, mcfg = bench.MODELS[model]
cfg = S.ModelConfig(**mcfg)
ids, offsets, lengths = newstest_corpus(bench.CORPUS, cfg.vocab_size)
eng = Engine(cfg, S.random_model(cfg, 0), dtype=dtype)
eng.reserve(3072, 64000)
dev = torch.device("cuda", 0)
L = lengths[:n]
b = budgets_of(L, 1.5, 5, cfg.max_positions)
off = np.zeros(n, np.int64)
np.cumsum(b[:-1], out=off[1:])
d_ids = torch.from_numpy(ids).to(dev)
d_off = torch.from_numpy(offsets[:n + 1]).to(dev)
d_out = torch.empty(int(b.sum()), dtype=torch.int32, device=dev)
d_oo = torch.from_numpy(off).to(dev)
d_len = torch.empty(n, dtype=torch.int32, device=dev)


def run():
    eng.translate_device(d_ids, d_off, L, d_out, off, d_oo, d_len, sbatch=3072, wbatch=64000,
                         beam=beam)


eng.profile(True)
run()                                   # warm (profiled path, same launch sequence)
torch.cuda.synchronize()
eng.profile(True)                       # reset the log
torch.cuda.profiler.start()
run()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
log = eng.profile_log()
eng.profile(False)
out = ROOT / "gpurun_out"
out.mkdir(exist_ok=True)
np.savez(out / f"prof_log_{tag}.npz", **log)
print("launches", len(log["cls"]), "words", int(d_len.sum()))
