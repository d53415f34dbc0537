"""CUDA-graph capture of the ops (launch-overhead probe): eager vs graph replay device time.  GPU tool."""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2601_18511_b200 import (HeContext, HeParams, encrypt_packed, make_mlwe_pcmm_plan, make_ring_pack_plan,
                                   make_slot_pcmm_plan, pcmm_level1, pcmm_mlwe, pcmm_slot_bsgs, ring_pack,
                                   ring_pack_keygen, slot_pcmm_keygen)
from paper_2601_18511_b200.rhombus import encrypt_vector, make_rhombus_plan, pcmv_rhombus, rhombus_keygen


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def graphed(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g.replay


P = HeParams.llama()
ctx = HeContext(P, rng="seeded")
sk = ctx.keygen(1)
rng = np.random.default_rng(0)
ops = {}
# Rhombus
keys = rhombus_keygen(ctx, sk, 3)
for n_out, n_in in ((4096, 11008), (14336, 4096)):
    W = rng.uniform(-1, 1, (n_out, n_in)) / math.sqrt(n_in)
    plan = make_rhombus_plan(ctx, W)
    x = encrypt_vector(ctx, sk, rng.uniform(-1, 1, n_in), seed=5)
    ops[f"rhombus {n_out}x{n_in}"] = (lambda plan=plan, x=x: pcmv_rhombus(ctx, plan, keys, x))
# slot PCMM
d = 128
sp = make_slot_pcmm_plan(ctx, rng.uniform(-1, 1, (d, d)) / math.sqrt(d))
sk_ = slot_pcmm_keygen(ctx, sk, sp, 7)
Xs = encrypt_packed(ctx, sk, rng.uniform(-1, 1, (d, d)), 1, seed=8)
ops["slot pcmm d=128"] = lambda: pcmm_slot_bsgs(ctx, sp, sk_, Xs)
# MLWE PCMM + ring pack
g = torch.Generator(device="cuda").manual_seed(1)
Wm = (torch.rand((4096, 11008), generator=g, device="cuda", dtype=torch.float64) * 2 - 1) / math.sqrt(11008)
A = torch.rand((P.tokens, 11008), generator=g, device="cuda", dtype=torch.float64) * 2 - 1
X = ctx.encrypt_acts(sk, A, seed=2)
pl = make_mlwe_pcmm_plan(ctx, Wm)
Y = pcmm_mlwe(ctx, pl, X)
ops["mlwe pcmm 4096x11008"] = lambda: pcmm_mlwe(ctx, pl, X, out=Y)
rk = ring_pack_keygen(ctx, sk, 9)
rp = make_ring_pack_plan(ctx, 4096)
rb, ra = pcmm_level1(ctx, pl, X, *rp.raw(ctx))
out = torch.empty((16, 1, 2, P.N), dtype=torch.int32, device="cuda")
ops["ring pack 4096"] = lambda: ring_pack(ctx, rp, rk, rb, ra, out)
for name, fn in ops.items():
    try:
        te = timed(fn)
        tg = timed(graphed(fn))
        print(f"{name}: eager {te:.3f} ms, graph {tg:.3f} ms", flush=True)
    except Exception as exc:
        print(f"{name}: graph capture failed: {exc!r}", flush=True)
