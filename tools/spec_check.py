"""Spectral (K7) vs direct (K1) MLWE PCMM: word equality, oracle parity on the toy ring, and
per-stage timing at a Llama shape.  Development tool (GPU)."""
import argparse
import math
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import oracle as O
from paper_2601_18511_b200 import HeContext, HeParams, make_mlwe_pcmm_plan, pcmm_mlwe

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="1024x4096,4096x11008")
ap.add_argument("--time", default="4096x11008")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()


def u32(t):
    return t.cpu().numpy().view(np.uint32)


# toy ring vs oracle
P = HeParams.toy()
ctx = HeContext(P, rng="seeded")
rng = np.random.default_rng(0)
for n_out, n_in in [(16, 16), (64, 48), (256, 384)]:
    A = rng.uniform(-1, 1, (P.tokens, n_in))
    W = rng.uniform(-1, 1, (n_out, n_in)) / np.sqrt(n_in)
    sk = ctx.keygen(7)
    X = ctx.encrypt_acts(sk, A, seed=11)
    ct = O.encrypt(P, 11, O.keygen(P, 7), O.encode_acts(P, A))
    ref = O.pcmm(P, O.encode_weights(P, W), ct)
    d, k = P.mlwe_degree, P.mlwe_rank
    for algo in ("direct", "spectral"):
        plan = make_mlwe_pcmm_plan(ctx, W, algo=algo)
        Y = pcmm_mlwe(ctx, plan, X)
        torch.cuda.synchronize()
        oa = u32(Y.out_a)
        ok_a = np.array_equal(oa, ref[:, d:])
        ob = u32(Y.out_b)
        ok_b = all(np.array_equal(ob[y // k, y % k + k * np.arange(d)], ref[y, :d]) for y in range(n_out))
        bad = int((oa != ref[:, d:]).sum())
        print(f"toy {n_out}x{n_in} {algo}: a' {'OK' if ok_a else 'MISMATCH'} ({bad} bad) b' {'OK' if ok_b else 'MISMATCH'}",
              flush=True)

P = HeParams.llama()
ctx = HeContext(P, rng="seeded")
g = torch.Generator(device="cuda").manual_seed(1)
for shp in a.shapes.split(","):
    n_out, n_in = (int(v) for v in shp.split("x"))
    W = (torch.rand((n_out, n_in), generator=g, device="cuda", dtype=torch.float64) * 2 - 1) / math.sqrt(n_in)
    A = torch.rand((P.tokens, n_in), generator=g, device="cuda", dtype=torch.float64) * 2 - 1
    sk = ctx.keygen(1)
    X = ctx.encrypt_acts(sk, A, seed=2)
    outs = {}
    for algo in ("direct", "spectral"):
        plan = make_mlwe_pcmm_plan(ctx, W, algo=algo)
        Y = pcmm_mlwe(ctx, plan, X)
        torch.cuda.synchronize()
        outs[algo] = (Y.out_a.clone(), Y.out_b.clone())
        if shp == a.time:
            st = torch.cuda.current_stream()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ts = []
            for _ in range(a.reps):
                ev[0].record()
                pcmm_mlwe(ctx, plan, X, out=Y)
                ev[1].record()
                torch.cuda.synchronize()
                ts.append(ev[0].elapsed_time(ev[1]))
            print(f"{shp} {algo}: {min(ts):.3f} ms/op (min of {a.reps}), median {sorted(ts)[len(ts)//2]:.3f}", flush=True)
        del plan
        torch.cuda.empty_cache()
    da = int((outs["direct"][0] != outs["spectral"][0]).sum())
    db = int((outs["direct"][1] != outs["spectral"][1]).sum())
    print(f"{shp}: spectral vs direct: a' mismatches {da}, b' mismatches {db}", flush=True)
    dec = ctx.decrypt_pcmm(sk, pcmm_mlwe(ctx, make_mlwe_pcmm_plan(ctx, W), X))
    ref = (A @ W.T).cpu().numpy()
    err = np.abs(dec - ref).max()
    print(f"{shp}: spectral decrypt max err {err:.3e} ({-math.log2(err / np.abs(ref).max()):.1f} bits rel)", flush=True)
