"""Ring packing (§8f1) at a Llama shape: device time of the level-1 PCMM, the packing, and the
end-to-end packed op (host input -> packed output on the host), plus decrypt precision.  GPU tool."""
import argparse
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2601_18511_b200 import (HeContext, HeParams, make_mlwe_pcmm_plan, make_ring_pack_plan, pcmm_level1,
                                   pcmm_mlwe, pcmm_packed, ring_pack, ring_pack_keygen)

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="4096x11008")
ap.add_argument("--reps", type=int, default=5)
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
Y = pcmm_packed(ctx, plan, rp, keys, X)
torch.cuda.synchronize()
dec = ctx.decrypt_acts(sk, Y)
ref = (A @ W.T).cpu().numpy()
err = np.abs(dec - ref).max()
print(f"{a.shape}: packed decrypt max err {err:.3e} ({-math.log2(err / np.abs(ref).max()):.1f} bits rel)", flush=True)


def timeit(fn):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for _ in range(a.reps):
        torch.cuda.synchronize()
        ev[0].record()
        fn()
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    return min(ts), sorted(ts)[len(ts) // 2]


raw_b, raw_a = rp.raw(ctx)
out = Y.data
t_l1 = timeit(lambda: pcmm_level1(ctx, plan, X, raw_b, raw_a))
t_rp = timeit(lambda: ring_pack(ctx, rp, keys, raw_b, raw_a, out))
t_all = timeit(lambda: pcmm_packed(ctx, plan, rp, keys, X, out))
Ym = pcmm_mlwe(ctx, plan, X)
t_mlwe = timeit(lambda: pcmm_mlwe(ctx, plan, X, out=Ym))
x_host = X.data.cpu().pin_memory()
y_host = torch.empty(out.shape, dtype=out.dtype).pin_memory()


def e2e():
    X.data.copy_(x_host, non_blocking=True)
    pcmm_packed(ctx, plan, rp, keys, X, out)
    y_host.copy_(out, non_blocking=True)


t_e2e = timeit(e2e)
ws = rp.workspace(ctx.device).numel() * 4
print(f"level-1 PCMM {t_l1[0]:.3f} ms | ring pack {t_rp[0]:.3f} ms | packed op {t_all[0]:.3f} ms "
      f"| MLWE op {t_mlwe[0]:.3f} ms | packed e2e {t_e2e[0]:.3f} ms (D2H {out.numel() * 4 / 1e6:.1f} MB) "
      f"| ring-pack ws {ws / 2**30:.2f} GiB", flush=True)
