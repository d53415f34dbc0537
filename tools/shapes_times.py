"""ms/op of the spectral and direct MLWE PCMM at every Llama projection shape (CUDA events).  Dev tool."""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2601_18511_b200 import HeContext, HeParams, make_mlwe_pcmm_plan, pcmm_mlwe

SHAPES = sys.argv[1].split(",") if len(sys.argv) > 1 else ["4096x4096", "4096x11008", "11008x4096", "14336x4096",
                                                            "4096x14336"]
ALGOS = sys.argv[2].split(",") if len(sys.argv) > 2 else ["spectral", "direct"]
P = HeParams.llama()
ctx = HeContext(P, rng="seeded")
g = torch.Generator(device="cuda").manual_seed(1)
for shp in SHAPES:
    n_out, n_in = (int(v) for v in shp.split("x"))
    W = (torch.rand((n_out, n_in), generator=g, device="cuda", dtype=torch.float64) * 2 - 1) / math.sqrt(n_in)
    A = torch.rand((P.tokens, n_in), generator=g, device="cuda", dtype=torch.float64) * 2 - 1
    X = ctx.encrypt_acts(ctx.keygen(1), A, seed=2)
    row = [shp]
    for algo in ALGOS:
        plan = make_mlwe_pcmm_plan(ctx, W, algo=algo)
        Y = pcmm_mlwe(ctx, plan, X)
        for _ in range(2):
            pcmm_mlwe(ctx, plan, X, out=Y)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10 if algo == "spectral" else 3
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            pcmm_mlwe(ctx, plan, X, out=Y)
        e1.record()
        torch.cuda.synchronize()
        row.append(f"{algo} {e0.elapsed_time(e1) / reps:.2f} ms")
        del plan, Y
        torch.cuda.empty_cache()
    print(" | ".join(row), flush=True)
