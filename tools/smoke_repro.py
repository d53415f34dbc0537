"""Repeat the smoke's PCMM + ring packing + SlotToCoeffs sequence in one process and fingerprint the StC inputs
(plan plaintexts, keys, input ct) and output each time, to locate an intermittent wrong StC result.  GPU tool."""
import hashlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import oracle as O
from paper_2601_18511_b200 import (HeContext, HeParams, make_mlwe_pcmm_plan, make_ring_pack_plan, pcmm_mlwe,
                                   pcmm_packed, ring_pack_keygen, slots)
from paper_2601_18511_b200.stc import (encrypt_slots, make_slot_to_coeffs_plan, slot_to_coeffs, slot_to_coeffs_keygen,
                                       slot_vectors)


def fp(t):
    return hashlib.md5(t.detach().cpu().numpy().tobytes()).hexdigest()[:8]


iters = int(sys.argv[1]) if len(sys.argv) > 1 else 10
P = HeParams.toy()
k = P.mlwe_rank
rng = np.random.default_rng(0)
n_out, n_in = 64, 48
A = rng.uniform(-1, 1, (P.tokens, n_in))
W = rng.uniform(-1, 1, (n_out, n_in)) / np.sqrt(n_in)
seen = {}
for it in range(iters):
    ctx = HeContext(P, rng="seeded")
    sk = ctx.keygen(7)
    X = ctx.encrypt_acts(sk, A, seed=11)
    for algo in ("spectral", "direct"):
        pcmm_mlwe(ctx, make_mlwe_pcmm_plan(ctx, W, algo=algo), X)
    pcmm_packed(ctx, make_mlwe_pcmm_plan(ctx, W), make_ring_pack_plan(ctx, n_out), ring_pack_keygen(ctx, sk, 5), X)
    sp = make_slot_to_coeffs_plan(ctx)
    keys = slot_to_coeffs_keygen(ctx, sk, sp, seed=17)
    Xs = encrypt_slots(ctx, sk, A[:, :k], seed=13, scale=sp.input_scale)
    Yc = slot_to_coeffs(ctx, sp, keys, Xs)
    torch.cuda.synchronize()
    f = {"pts": fp(sp.pts), "keys": "/".join(fp(getattr(keys, a)) for a in sorted(vars(keys))
                                              if torch.is_tensor(getattr(keys, a))),
         "x": fp(Xs.data), "out": fp(Yc.data[0, 0])}
    print(it, f, flush=True)
    for kk, v in f.items():
        seen.setdefault(kk, set()).add(v)
print({kk: len(v) for kk, v in seen.items()})
