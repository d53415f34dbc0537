"""One warm-up + one profiled Rhombus PCMv (for ncu launch lists)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2601_18511_b200 import HeContext, HeParams, encrypt_vector, make_rhombus_plan, pcmv_rhombus, rhombus_keygen

n_out, n_in = (int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "4096x11008").split("x"))
P = HeParams.llama()
ctx = HeContext(P, rng="seeded")
sk = ctx.keygen(7)
keys = rhombus_keygen(ctx, sk, 99)
rng = np.random.default_rng(1)
x = encrypt_vector(ctx, sk, rng.uniform(-1, 1, n_in), seed=5)
plan = make_rhombus_plan(ctx, rng.uniform(-1, 1, (n_out, n_in)) / np.sqrt(n_in))
for _ in range(2):
    y = pcmv_rhombus(ctx, plan, keys, x)
torch.cuda.synchronize()
print("done")
