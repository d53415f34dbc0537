"""The GPU slot-domain PCMM in the reference's PC-attention flow: scores and values
products on ciphertexts (shear chain 2 -> 1 -> 0), RoPE and softmax on the key holder's side, against
the reference's clear oracle (clear_pc_attention, golden values from hesim)."""
from pathlib import Path

import numpy as np
import pytest

from paper_2601_18511_b200 import HeContext, HeParams
from paper_2601_18511_b200.attention import clear_pc_attention, pc_attention_hybrid

pytestmark = pytest.mark.gpu
G = np.load(Path(__file__).parent / "golden" / "attention_golden.npz")


@pytest.mark.parametrize("d,params,tol", [(8, "toy", 1e-4), (16, "toy", 1e-4), (64, "llama", 5e-3)])
def test_pc_attention_hybrid_matches_hesim_oracle(d, params, tol):
    q, k, v, ref = G[f"d{d}_q"], G[f"d{d}_k"], G[f"d{d}_v"], G[f"d{d}_out"]
    positions = d + np.arange(d)
    np.testing.assert_allclose(clear_pc_attention(q, k, v, positions), ref, atol=1e-12)   # restatement
    P = HeParams.toy() if params == "toy" else HeParams.llama()
    ctx = HeContext(P, rng="seeded")
    sk = ctx.keygen(3)
    out, rep = pc_attention_hybrid(ctx, sk, q, k, v, positions, seed=10)
    assert rep["ledger"]["rescales"] == 2
    assert np.abs(out - ref).max() < tol, np.abs(out - ref).max()


@pytest.mark.parametrize("d,params,tol", [(8, "toy", 1e-4), (16, "toy", 1e-4), (64, "llama", 2e-3)])
def test_rope_packed_matches_hesim(d, params, tol):
    """hesim rope_packed (one rotation + a 2-term pc_linear, one level) as a GPU slot linear map on a
    twice-sheared ciphertext, against hesim's own rope_packed values."""
    from paper_2601_18511_b200.slotpcmm import decrypt_packed, encrypt_packed, make_rope_plan, slot_linear, \
        slot_linear_keygen

    q, ref = G[f"d{d}_q"], G[f"d{d}_rope2"]
    positions = d + np.arange(d)
    P = HeParams.toy() if params == "toy" else HeParams.llama()
    ctx = HeContext(P, rng="seeded")
    sk = ctx.keygen(3)
    plan = make_rope_plan(ctx, d, positions, shear_power=2)
    keys = slot_linear_keygen(ctx, sk, plan, seed=4)
    before = ctx.ledger.snapshot()
    Y = slot_linear(ctx, plan, keys, encrypt_packed(ctx, sk, q, 2, seed=5))
    led = ctx.ledger.diff(before)
    assert led["ct_rotations"] == 1 and led["rescales"] == 1 and Y.level == 0 and Y.shear_power == 2
    # N = 2^16: the masks are slot-encoded at scale q1 = 2^20.2, i.e. ~2^-14 per slot (the slot-encoding bound)
    assert np.abs(decrypt_packed(ctx, sk, Y) - ref).max() < tol
