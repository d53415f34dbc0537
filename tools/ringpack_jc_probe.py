"""Ring-pack pass size (HE_MS_JC) eager vs CUDA-graph replay.  GPU tool (run once per HE_MS_JC value)."""
import math
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2601_18511_b200 import (HeContext, HeParams, OpGraph, make_mlwe_pcmm_plan, make_ring_pack_plan,
                                   pcmm_level1, ring_pack, ring_pack_keygen)

P = HeParams.llama()
ctx = HeContext(P, rng="seeded")
sk = ctx.keygen(1)
g = torch.Generator(device="cuda").manual_seed(1)
W = (torch.rand((4096, 11008), generator=g, device="cuda", dtype=torch.float64) * 2 - 1) / math.sqrt(11008)
A = torch.rand((P.tokens, 11008), generator=g, device="cuda", dtype=torch.float64) * 2 - 1
X = ctx.encrypt_acts(sk, A, seed=2)
pl = make_mlwe_pcmm_plan(ctx, W)
rk = ring_pack_keygen(ctx, sk, 9)
rp = make_ring_pack_plan(ctx, 4096)
rb, ra = pcmm_level1(ctx, pl, X, *rp.raw(ctx))
out = torch.empty((16, 1, 2, P.N), dtype=torch.int32, device="cuda")


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


fn = lambda: ring_pack(ctx, rp, rk, rb, ra, out)  # noqa: E731
print(f"jc={os.environ.get('HE_MS_JC', 'default')}: eager {timed(fn):.3f} ms, graph {timed(OpGraph(fn).replay):.3f} ms",
      flush=True)
