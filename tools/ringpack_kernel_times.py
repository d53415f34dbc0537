"""Per-kernel device times of ring packing (keyswitch1) at a Llama shape in a normal run (torch.profiler /
CUPTI), averaged over reps.  GPU tool."""
import argparse
import collections
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2601_18511_b200 import (HeContext, HeParams, make_mlwe_pcmm_plan, make_ring_pack_plan, pcmm_level1,
                                   ring_pack, ring_pack_keygen)

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="4096x11008")
ap.add_argument("--method", default="keyswitch1")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
n_out, n_in = (int(v) for v in a.shape.split("x"))
P = HeParams.llama()
ctx = HeContext(P, rng="seeded")
g = torch.Generator(device="cuda").manual_seed(1)
W = (torch.rand((n_out, n_in), generator=g, device="cuda", dtype=torch.float64) * 2 - 1) / math.sqrt(n_in)
A = torch.rand((P.tokens, n_in), generator=g, device="cuda", dtype=torch.float64) * 2 - 1
sk = ctx.keygen(1)
X = ctx.encrypt_acts(sk, A, seed=2)
keys = ring_pack_keygen(ctx, sk, seed=3, method=a.method)
plan = make_mlwe_pcmm_plan(ctx, W)
rp = make_ring_pack_plan(ctx, n_out, method=a.method)
raw_b, raw_a = pcmm_level1(ctx, plan, X, *rp.raw(ctx))
for _ in range(2):
    ring_pack(ctx, rp, keys, raw_b, raw_a)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    ev[0].record()
    for _ in range(a.reps):
        ring_pack(ctx, rp, keys, raw_b, raw_a)
    ev[1].record()
    torch.cuda.synchronize()
tot = collections.defaultdict(float)
cnt = collections.Counter()
for e in prof.events():
    if e.device_type.name == "CUDA":
        tot[e.name[:70]] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
        cnt[e.name[:70]] += 1
print(f"{a.shape} ring pack ({a.method}): {ev[0].elapsed_time(ev[1]) / a.reps:.3f} ms (events, {a.reps} reps)")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"  {v / a.reps / 1000:8.3f} ms  x{cnt[k] // a.reps}  {k}")
