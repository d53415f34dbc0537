"""One warm-up + one profiled MLWE PCMM op at a Llama shape (for ncu captures; no timing)."""
import argparse
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2601_18511_b200 import HeContext, HeParams, make_mlwe_pcmm_plan, pcmm_mlwe

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="4096x11008")
ap.add_argument("--ops", type=int, default=2)
ap.add_argument("--algo", default="spectral")
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
for _ in range(a.ops):
    Y = pcmm_mlwe(ctx, plan, X)
torch.cuda.synchronize()
print("done", plan.d_w)
