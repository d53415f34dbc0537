"""Per-kernel device times of one Rhombus PCMv op (torch.profiler / CUPTI).  Development tool (GPU)."""
import collections
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2601_18511_b200 import HeContext, HeParams, encrypt_vector, make_rhombus_plan, pcmv_rhombus, rhombus_keygen

for shape in (sys.argv[1:] or ["4096x11008", "14336x4096"]):
    n_out, n_in = (int(v) for v in shape.split("x"))
    P = HeParams.llama()
    ctx = HeContext(P, rng="seeded")
    sk = ctx.keygen(7)
    keys = rhombus_keygen(ctx, sk, 99)
    rng = np.random.default_rng(1)
    x = encrypt_vector(ctx, sk, rng.uniform(-1, 1, n_in), seed=5)
    plan = make_rhombus_plan(ctx, rng.uniform(-1, 1, (n_out, n_in)) / np.sqrt(n_in))
    for _ in range(2):
        pcmv_rhombus(ctx, plan, keys, x)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile

    ops = 3
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(ops):
            pcmv_rhombus(ctx, plan, keys, x)
        torch.cuda.synchronize()
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for e in prof.events():
        if e.device_type.name == "CUDA":
            tot[e.name[:70]] += e.device_time_total
            cnt[e.name[:70]] += 1
    print(f"{shape}: total {sum(tot.values()) / ops / 1000:.3f} ms/op (sum of kernels)")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:14]:
        print(f"  {v / ops / 1000:8.3f} ms  x{cnt[k] // ops:4d}  {k}")
