"""SlotToCoeffs precision at N = 2^16 against the plaintext scale split (pt_shift): plaintexts at q1 2^t,
input slots at Delta / 2^t.  GPU tool."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2601_18511_b200 import HeContext, HeParams
from paper_2601_18511_b200.stc import encrypt_slots, make_slot_to_coeffs_plan, slot_to_coeffs, slot_to_coeffs_keygen

ctx = HeContext(HeParams.llama(), rng="seeded")
sk = ctx.keygen(1)
P = ctx.params
n = P.N // 2
A = np.random.default_rng(0).uniform(-1, 1, (P.mlwe_degree // 2, P.mlwe_rank))
lazy = "--lazy" in sys.argv
for t in [int(v) for v in sys.argv[1:] if v != "--lazy"] or [0, 2, 4, 6]:
    plan = make_slot_to_coeffs_plan(ctx, pt_shift=t, lazy=lazy)
    keys = slot_to_coeffs_keygen(ctx, sk, plan, seed=2)
    X = encrypt_slots(ctx, sk, A, seed=3, scale=plan.input_scale)
    Y = slot_to_coeffs(ctx, plan, keys, X)
    ph = ctx.decrypt_phase(sk, Y).cpu().numpy()[0].astype(float) / P.delta
    err = np.abs(ctx.decrypt_acts(sk, Y) - A)
    print(f"{'lazy ' if lazy else ''}pt_shift {t}: max err {err.max():.2e} ({-np.log2(err.max()):.1f} bits), rms {np.sqrt((err ** 2).mean()):.2e}, "
          f"imag half max {np.abs(ph[n:]).max():.2e}", flush=True)
    del plan, keys, X, Y
    torch.cuda.empty_cache()
