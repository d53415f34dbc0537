"""CoeffToSlots precision at N = 2^16 on a ModRaised level-0 ciphertext, against the integer pre-multiplication
and the per-map plaintext scale shifts (chain.make_factorized_cts_plan).  python tools/cts_precision.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

import oracle as O
from paper_2601_18511_b200 import HeContext, HeParams, mod_raise, slots
from paper_2601_18511_b200.chain import (coeffs_to_slots_factorized, decrypt_exact, encrypt_coeffs_at,
                                         factorized_stc_keygen, make_factorized_cts_plan)
from paper_2601_18511_b200.context import CtBlocks
from paper_2601_18511_b200.stc import slot_of_coeff

P = HeParams.llama_chain(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
ctx = HeContext(P, rng="seeded")
sk = ctx.keygen(7)
A = np.random.default_rng(5).uniform(-1, 1, (P.tokens, P.mlwe_rank))
X0 = encrypt_coeffs_at(ctx, sk, O.encode_acts(P, A), level=0, seed=3)
raised = mod_raise(ctx, CtBlocks(X0.data, level=0, n_cols=0), list(P.moduli))
ph = np.asarray(decrypt_exact(ctx, sk, raised), dtype=np.float64)
c = np.argsort(slot_of_coeff(P.N))
want = ph[:, c] + 1j * ph[:, P.N // 2 + c]
CFG = [(0, None), (0, (0, 0, 0)), (0, (-6, -6, -6)), (6, (-4, -4, -4)), (0, (-8, -8, 0))]
if P.top_level >= 5:
    CFG += [(0, (-10, -10, -10)), (0, (-12, -12, -12)), (0, (-15, -15, -15)), (8, (-12, -12, -12))]
for pre, sh in CFG:
    plan = make_factorized_cts_plan(ctx, shifts=sh, pre_log2=pre)
    keys = factorized_stc_keygen(ctx, sk, plan, seed=9)
    Z = coeffs_to_slots_factorized(ctx, plan, keys, raised)
    out = np.asarray(decrypt_exact(ctx, sk, Z.data), dtype=np.float64)
    got = np.stack([slots.decode(v, P.N, Z.scale, real=False) for v in out])
    err = np.abs(got - want).max()
    print(f"top level {P.top_level} pre {pre:2d} shifts {plan.shifts} (given {sh}): err 2^{np.log2(err / P.moduli[0]):6.1f} q0, output |coef| <= "
          f"2^{np.log2(np.abs(out).max()):.1f} (q0 q1 / 2 = 2^{np.log2(P.moduli[0] * P.moduli[1] / 2):.1f})", flush=True)
