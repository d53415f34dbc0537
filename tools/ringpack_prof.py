"""One ring-pack run at a Llama shape after a warm-up, for ncu launch lists.  GPU tool."""
import argparse
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2601_18511_b200 import (HeContext, HeParams, make_mlwe_pcmm_plan, make_ring_pack_plan, pcmm_level1,
                                   ring_pack, ring_pack_keygen)

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="4096x11008")
ap.add_argument("--method", default="keyswitch")
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
ring_pack(ctx, rp, keys, raw_b, raw_a)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
ring_pack(ctx, rp, keys, raw_b, raw_a)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
