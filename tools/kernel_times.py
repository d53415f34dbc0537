"""Per-kernel device times of the MLWE PCMM op in a normal (unprofiled-by-ncu) run, via the
CUDA profiler activity API (torch.profiler / CUPTI).  Development tool (GPU)."""
import argparse
import collections
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2601_18511_b200 import HeContext, HeParams, make_mlwe_pcmm_plan, pcmm_mlwe

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="4096x11008")
ap.add_argument("--algo", default="spectral")
ap.add_argument("--ops", type=int, default=5)
a = ap.parse_args()
n_out, n_in = (int(v) for v in a.shape.split("x"))
P = HeParams.llama()
ctx = HeContext(P, rng="seeded")
g = torch.Generator(device="cuda").manual_seed(1)
W = (torch.rand((n_out, n_in), generator=g, device="cuda", dtype=torch.float64) * 2 - 1) / math.sqrt(n_in)
A = torch.rand((P.tokens, n_in), generator=g, device="cuda", dtype=torch.float64) * 2 - 1
sk = ctx.keygen(1)
X = ctx.encrypt_acts(sk, A, seed=2)
plan = make_mlwe_pcmm_plan(ctx, W, algo=a.algo)
Y = pcmm_mlwe(ctx, plan, X)
Y = pcmm_mlwe(ctx, plan, X, out=Y)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile

ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    ev[0].record()
    for _ in range(a.ops):
        pcmm_mlwe(ctx, plan, X, out=Y)
    ev[1].record()
    torch.cuda.synchronize()
tot = collections.defaultdict(float)
cnt = collections.Counter()
for e in prof.events():
    if e.device_type.name == "CUDA":
        tot[e.name[:80]] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
        cnt[e.name[:80]] += 1
print(f"{a.shape} {a.algo}: {ev[0].elapsed_time(ev[1]) / a.ops:.3f} ms/op (events, {a.ops} ops)")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"  {v / a.ops / 1000:8.3f} ms/op  x{cnt[k] // a.ops}  {k}")
