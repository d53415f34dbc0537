"""Repeat the smoke's toy SlotToCoeffs check (fresh keys / plan / ciphertexts each iteration, same seeds) and
report any iteration whose words differ from the oracle.  GPU tool (investigating an intermittent smoke failure)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import oracle as O
from paper_2601_18511_b200 import HeContext, HeParams, slots
from paper_2601_18511_b200.stc import (encrypt_slots, make_slot_to_coeffs_plan, slot_to_coeffs, slot_to_coeffs_keygen,
                                       slot_vectors, stc_plaintexts)

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
P = HeParams.toy()
rng = np.random.default_rng(0)
k = P.mlwe_rank
A = rng.uniform(-1, 1, (P.tokens, 48))
bad = 0
ref_sc = None
for it in range(iters):
    ctx = HeContext(P, rng="seeded")
    sk = ctx.keygen(7)
    sp = make_slot_to_coeffs_plan(ctx)
    b, g, n = sp.split.baby, sp.split.giant, P.N // 2
    keys = slot_to_coeffs_keygen(ctx, sk, sp, seed=17)
    Xs = encrypt_slots(ctx, sk, A[:, :k], seed=13, scale=sp.input_scale)
    Yc = slot_to_coeffs(ctx, sp, keys, Xs)
    torch.cuda.synchronize()
    if ref_sc is None:
        s = O.keygen(P, 7)
        cs = O.encrypt(P, 13, s, slots.encode(slot_vectors(P, A[:, :k])[0], P.N, sp.input_scale)[None])[0]
        pt = stc_plaintexts(P, sp.split, 0, n, pt_shift=sp.pt_shift).numpy()
        pts = np.stack([np.stack([(pt[t] % q).astype(np.uint32) for q in P.ks_moduli]) for t in range(n)])
        ref_sc = O.slot_bsgs(P, cs, pts, 1, b, g, O.rotation_keys(P, 17, s, list(range(1, b))),
                             O.rotation_keys_plain(P, 17, s, [j * b for j in range(1, g)]), lazy=True)
    got = Yc.data.cpu().numpy().view(np.uint32)[0, 0]
    if not np.array_equal(got, ref_sc):
        bad += 1
        dif = np.argwhere(got != ref_sc)
        print(f"iter {it}: {len(dif)} words differ, first {dif[:5].tolist()}", flush=True)
        # which stage: keys or ciphertext?
        xs_ref = O.encrypt(P, 13, O.keygen(P, 7), slots.encode(slot_vectors(P, A[:, :k])[0], P.N, sp.input_scale)[None])[0]
        print("  input ct equal:", np.array_equal(Xs.data.cpu().numpy().view(np.uint32)[0], xs_ref), flush=True)
print(f"{bad} of {iters} iterations differ")
